// online_lse.cuh — the online log-sum-exp / entropy / KL accumulation over
// bf16 logit vectors shared by A1 (token_stats.cu) and the fused loss +
// gradient kernel (policy_loss_grad.cu): log2-domain accumulators with
// integer bases (rebases are exact powers of two), packed f32x2 math, the
// bf16x2 max / floor helpers and the thread -> warp -> CTA combine of row
// partials.  Numerics follow the reference's max-subtracted softmax
// (proj/src/distattn.cpp:99-123) in one pass with an online maximum.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace yattb {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLn2 = 0.69314718055994530942;
constexpr float kLn2f = 0.69314718f;
constexpr float kSlack = 24.0f;  // allow 2^a up to 2^24 before re-basing
constexpr int kMinitial = -(1 << 24);
constexpr uint32_t kNegInf2 = 0xFF80FF80u;  // two bf16 -inf

// Words (bf16 pairs) of each 8-element vector whose 2^a goes through the FMA
// pipe (polynomial) instead of MUFU.EX2, per tensor: balances the MUFU pipe
// (16 ex2/clk/SM) against the issue port.  0 = all MUFU.
#ifndef YATT_A1_POLY_WORDS
#define YATT_A1_POLY_WORDS 0
#endif
constexpr int kPolyWords = YATT_A1_POLY_WORDS;

struct RowPartial {
  float mp, s, w, mq, sq, u;
};

// Per-thread online state for one row.  Element pairs (the two bf16 of one
// 32-bit word) are processed with Blackwell's packed f32x2 FMA/ADD
// (FFMA2/FADD2: two IEEE fp32 RN operations per instruction), halving the
// FMA-pipe issue count; each lane keeps the exact per-element arithmetic.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
// 2^a on the FMA pipe for a pair: Cody-Waite split a = n + r (|r| <= 1/2)
// with the 1.5*2^23 rounding trick, degree-5 near-minimax polynomial for
// 2^r (max rel err 2.3e-7 in fp32, same class as ex2.approx), exponent
// inserted with one integer multiply-add.  a is clamped to >= -125 so the
// exponent insertion cannot wrap (2^-125 ~ 0 for masked-vocab logits).
__device__ __forceinline__ float2 ex2_poly2(float2& a) {
  a = f2(fmaxf(a.x, -125.f), fmaxf(a.y, -125.f));
  const float2 magic = f2(12582912.f, 12582912.f);
  const float2 j = __fadd2_rn(a, magic);
  const float2 n = __fadd2_rn(j, f2(-12582912.f, -12582912.f));
  const float2 r = __ffma2_rn(n, f2(-1.f, -1.f), a);
  float2 p = __ffma2_rn(f2(0.001327647129073739f, 0.001327647129073739f), r,
                        f2(0.009675541892647743f, 0.009675541892647743f));
  p = __ffma2_rn(p, r, f2(0.05550713092088699f, 0.05550713092088699f));
  p = __ffma2_rn(p, r, f2(0.24022120237350464f, 0.24022120237350464f));
  p = __ffma2_rn(p, r, f2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(p, r, f2(1.0000001192092896f, 1.0000001192092896f));
  return f2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(j.x) << 23)),
            __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(j.y) << 23)));
}

__device__ __forceinline__ float2 ex2x2(float2 a) {
  return make_float2(ex2_approx(a.x), ex2_approx(a.y));
}

// kRef = false: policy only (no reference logits; the fused loss + gradient
// kernel), the q accumulators stay empty.
template <bool kFull, bool kRef = true>
struct Acc {
  float2 s[4], w[4], sq[4], u[4];
  float mp, mq;        // integer-valued bases (log2 units)
  float thr_p, thr_q;  // rebase when a logit exceeds these

  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      s[k] = w[k] = sq[k] = f2(0.f, 0.f);
      if (kFull) u[k] = f2(0.f, 0.f);
    }
    mp = mq = float(kMinitial);
    thr_p = thr_q = (float(kMinitial) + kSlack) * kLn2f;
  }

  // Rebase policy accumulators to m' = ceil(vmax*log2e): exact 2^(m-m').
  __device__ __forceinline__ void rebase_p(float vmax) {
    float mn = ceilf(vmax * kLog2e);
    mn = fminf(fmaxf(mn, float(kMinitial)), float(1 << 24));
    if (mn <= mp) return;
    const float d = mp - mn;
    const float c = exp2_int(int(d));
    const float2 c2 = f2(c, c), d2 = f2(d, d);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      w[k] = __fmul2_rn(c2, __ffma2_rn(d2, s[k], w[k]));
      s[k] = __fmul2_rn(c2, s[k]);
      if (kFull) u[k] = __fmul2_rn(c2, u[k]);
    }
    mp = mn;
    thr_p = (mp + kSlack) * kLn2f;
  }
  __device__ __forceinline__ void rebase_q(float vmax) {
    float mn = ceilf(vmax * kLog2e);
    mn = fminf(fmaxf(mn, float(kMinitial)), float(1 << 24));
    if (mn <= mq) return;
    const float c = exp2_int(int(mq - mn));
#pragma unroll
    for (int k = 0; k < 4; ++k) sq[k] = __fmul2_rn(f2(c, c), sq[k]);
    mq = mn;
    thr_q = (mq + kSlack) * kLn2f;
  }

  // Accumulate one 8-element vector pair (policy P already floored).
  __device__ __forceinline__ void step(const uint4& P, const uint4& Q) {
    const uint32_t pw[4] = {P.x, P.y, P.z, P.w};
    const uint32_t qw[4] = {Q.x, Q.y, Q.z, Q.w};
    const float2 L2 = f2(kLog2e, kLog2e);
    const float2 nmp = f2(-mp, -mp), nmq = f2(-mq, -mq);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 x = f2(bf16_lo(pw[k]), bf16_hi(pw[k]));
      const float2 z = f2(bf16_lo(qw[k]), bf16_hi(qw[k]));
      const float2 a = __ffma2_rn(x, L2, nmp);
      float2 a_used = a;
      const float2 e = k < kPolyWords ? ex2_poly2(a_used) : ex2x2(a);
      s[k] = __fadd2_rn(s[k], e);
      w[k] = __ffma2_rn(e, a_used, w[k]);
      if (kRef) {
        const float2 b = __ffma2_rn(z, L2, nmq);
        float2 b_used = b;
        sq[k] = __fadd2_rn(sq[k], k < kPolyWords ? ex2_poly2(b_used) : ex2x2(b));
      }
      if (kFull) u[k] = __ffma2_rn(e, __ffma2_rn(z, f2(-1.f, -1.f), x), u[k]);
    }
  }

  // Thread total of one accumulator set (pairwise tree).
  __device__ __forceinline__ static float total(const float2 (&v)[4]) {
    return ((v[0].x + v[0].y) + (v[1].x + v[1].y)) + ((v[2].x + v[2].y) + (v[3].x + v[3].y));
  }
};

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a),
                             *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t vmax4(const uint4& v) {
  return bmax2(bmax2(v.x, v.y), bmax2(v.z, v.w));
}
__device__ __forceinline__ float pair_max(uint32_t m2) {
  return fmaxf(bf16_lo(m2), bf16_hi(m2));
}
// Floor the policy logits at -1e30 (bf16 0xF149): keeps 2^a * a finite for
// -inf (masked-vocab) logits; exact for every finite logit above it.
__device__ __forceinline__ uint4 floor_policy(uint4 v) {
  constexpr uint32_t kFloor = 0xF149F149u;
  v.x = bmax2(v.x, kFloor);
  v.y = bmax2(v.y, kFloor);
  v.z = bmax2(v.z, kFloor);
  v.w = bmax2(v.w, kFloor);
  return v;
}

// Keep elements [lo, hi) of an 8-element bf16 vector, -inf elsewhere (row
// edges of an aligned staging superset when V % 8 != 0).
__device__ __forceinline__ uint4 keep_range(uint4 v, int lo, int hi) {
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (2 * k < lo || 2 * k >= hi) w[k] = (w[k] & 0xffff0000u) | 0xFF80u;
    if (2 * k + 1 < lo || 2 * k + 1 >= hi) w[k] = (w[k] & 0x0000ffffu) | 0xFF800000u;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ RowPartial combine(const RowPartial& A, const RowPartial& B) {
  RowPartial r;
  r.mp = fmaxf(A.mp, B.mp);
  {
    const float da = A.mp - r.mp, db = B.mp - r.mp;
    const float ca = exp2_int(int(da)), cb = exp2_int(int(db));
    r.s = ca * A.s + cb * B.s;
    r.w = ca * fmaf(da, A.s, A.w) + cb * fmaf(db, B.s, B.w);
    r.u = ca * A.u + cb * B.u;
  }
  r.mq = fmaxf(A.mq, B.mq);
  r.sq = exp2_int(int(A.mq - r.mq)) * A.sq + exp2_int(int(B.mq - r.mq)) * B.sq;
  return r;
}

__device__ __forceinline__ RowPartial shfl_partial(const RowPartial& p, int off) {
  RowPartial o;
  o.mp = __shfl_xor_sync(0xffffffffu, p.mp, off);
  o.s = __shfl_xor_sync(0xffffffffu, p.s, off);
  o.w = __shfl_xor_sync(0xffffffffu, p.w, off);
  o.mq = __shfl_xor_sync(0xffffffffu, p.mq, off);
  o.sq = __shfl_xor_sync(0xffffffffu, p.sq, off);
  o.u = __shfl_xor_sync(0xffffffffu, p.u, off);
  return o;
}

// Warp-wide combine: butterfly max of the integer bases, ONE exact
// power-of-two rescale per thread, then plain butterfly sums (instead of five
// pairwise combines that each rescale both sides).  Result on all lanes.
template <bool kFull>
__device__ __forceinline__ RowPartial warp_combine(RowPartial r) {
  float Mp = r.mp, Mq = r.mq;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Mp = fmaxf(Mp, __shfl_xor_sync(0xffffffffu, Mp, off));
    Mq = fmaxf(Mq, __shfl_xor_sync(0xffffffffu, Mq, off));
  }
  const float d = r.mp - Mp;
  const float c = exp2_int(int(d));
  float s = c * r.s, w = c * fmaf(d, r.s, r.w), u = kFull ? c * r.u : 0.f;
  float sq = exp2_int(int(r.mq - Mq)) * r.sq;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, off);
    w += __shfl_xor_sync(0xffffffffu, w, off);
    sq += __shfl_xor_sync(0xffffffffu, sq, off);
    if (kFull) u += __shfl_xor_sync(0xffffffffu, u, off);
  }
  return RowPartial{Mp, s, w, Mq, sq, u};
}

// Re-base a thread's partial so its sum lies in [1, 2): makes the cross-
// thread combine safe even when the fast path let a thread's terms grow far
// above (or below) its base.  Exact (power-of-two scaling).
__device__ __forceinline__ RowPartial normalize(RowPartial r) {
  if (r.s > 0.f && r.s <= 3.4e38f) {
    const int k = ilogbf(r.s);
    r.w = ldexpf(fmaf(-float(k), r.s, r.w), -k);
    r.s = ldexpf(r.s, -k);
    r.u = ldexpf(r.u, -k);
    r.mp += float(k);
  }
  if (r.sq > 0.f && r.sq <= 3.4e38f) {
    const int k = ilogbf(r.sq);
    r.sq = ldexpf(r.sq, -k);
    r.mq += float(k);
  }
  return r;
}

template <bool kFull>
__device__ __forceinline__ bool partial_finite(const RowPartial& q) {
  return isfinite(q.s) && isfinite(q.w) && isfinite(q.sq) && (!kFull || isfinite(q.u)) &&
         q.s > 0.f && q.sq > 0.f;
}

}  // namespace
}  // namespace yattb
