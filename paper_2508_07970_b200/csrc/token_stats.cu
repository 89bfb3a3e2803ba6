// token_stats.cu — A1: fused single-pass log-prob / entropy / KL over bf16
// policy and reference logits.
//
// Replaces the Preparation-stage cost stand-in of the reference
// (proj/src/simcore.cpp:13-15, :395-398: "policy and reference policy compute
// their reference log probabilities") with the real per-token
// computation.  Numerics follow the reference's max-subtracted softmax
// (proj/src/distattn.cpp:99-123) but in ONE pass with an online maximum.
//
// Layout: policy / ref logits are row-major [rows, V] bf16, one row per token.
// Bound: HBM.  Algorithmic bytes per valid row = 4V (two bf16 rows) + 4
// (target) + 1 (mask) + 16 (four fp32 outputs) = 4V + 21.
//
// Kernel structure (persistent, warp-specialised, 2 CTAs per SM):
//   warp 8      : producer — one elected lane streams each row in TILE-element
//                 pieces of both tensors into a STAGES-deep shared-memory ring
//                 with cp.async.bulk (TMA bulk engine), completion tracked by
//                 mbarrier transaction counts; L2 evict-first policy.
//   warps 0..7  : consumers — 128-bit ld.shared of 8 bf16 per tensor per
//                 step, online log-sum-exp in the log2 domain:
//                   a = x*log2e - m   (m integer: rescales are exact 2^k)
//                   s += 2^a ; w += 2^a * a        (policy: lse + entropy)
//                   sq += 2^b                      (reference: lse)
//                   u += 2^a (x - z)               (FULL KL only)
//                 8 independent accumulators per quantity per thread (short
//                 fp32 chains), warp-shuffle + smem combine at row end, fp64
//                 epilogue by a rotating warp.  The target logits are picked
//                 out of the staged tile by whichever thread holds them — no
//                 extra global loads.
// Any vocab on 16-byte-aligned tensors: with V % 8 != 0 (kEdges) each row is
// staged as its aligned superset (up to 7 neighbouring elements per side),
// the edge vectors masked to -inf; the last row takes the generic kernel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "grad_math.cuh"

namespace yattb {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;  // + producer warp
#ifdef YATT_A1_SMALL_TU  // token_stats_small.cu: the ring shape for small vocabularies
#define YATT_A1_TILE YATT_A1_SMALL_TILE
#define YATT_A1_STAGES YATT_A1_SMALL_STAGES
#define YATT_A1_MINB YATT_A1_SMALL_MINB
#endif
#ifndef YATT_A1_TILE
#define YATT_A1_TILE 8192
#endif
#ifndef YATT_A1_STAGES
#define YATT_A1_STAGES 3
#endif
#ifndef YATT_A1_MINB
#define YATT_A1_MINB 2
#endif
constexpr int kTile = YATT_A1_TILE;        // bf16 elements per tensor per stage
constexpr int kStages = YATT_A1_STAGES;
constexpr int kMinBlocks = YATT_A1_MINB;   // resident CTAs per SM (grid = kMinBlocks x SMs)
constexpr int kVecPerTile = kTile / 8;                  // 16-byte vectors
constexpr int kVecPerThread = kVecPerTile / kConsumers;  // full-tile unroll
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLn2 = 0.69314718055994530942;
constexpr float kLn2f = 0.69314718f;
constexpr float kSlack = 24.0f;  // allow 2^a up to 2^24 before re-basing
constexpr int kMinitial = -(1 << 24);
// Words (bf16 pairs) of each 8-element vector whose 2^a goes through the FMA
// pipe (polynomial) instead of MUFU.EX2, per tensor: balances the MUFU pipe
// (16 ex2/clk/SM) against the issue port.  0 = all MUFU.
#ifndef YATT_A1_POLY_WORDS
#define YATT_A1_POLY_WORDS 0
#endif
constexpr int kPolyWords = YATT_A1_POLY_WORDS;
static_assert(kVecPerTile % kConsumers == 0, "tile must split evenly");

struct RowPartial {
  float mp, s, w, mq, sq, u;
};

struct __align__(16) SmemTail {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  RowPartial red[2][kConsumerWarps];
  float tgt[2][2];
};

constexpr size_t kRingBytes = size_t(kStages) * 2 * kTile * sizeof(uint16_t);
constexpr size_t kSmemBytes = kRingBytes + sizeof(SmemTail);

}  // namespace

// Shared by token_stats.cu and token_stats_small.cu (same definition).
struct A1Params {
  const uint16_t* pol;
  const uint16_t* ref;
  const int32_t* tgt;
  const uint8_t* mask;
  int64_t rows;
  int32_t V;
  int32_t kl_mode;
  float* logp;
  float* ref_logp;
  float* ent;
  float* kl;
};

namespace {


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

// Per-thread normalisation before the warp combine (s into [1, 2)).  With
// the max-of-bases combine it only changes where an overflow is caught (an
// infinite lane sum is flagged for the fix-up kernel either way); off by
// default: V=32000 5.53 -> 5.78 TB/s, V=8192 3.15 -> 3.50 TB/s.
#ifndef YATT_A1_NORMALIZE
#define YATT_A1_NORMALIZE 0
#endif

#ifndef YATT_A1_FASTPATH
#define YATT_A1_FASTPATH 1
#endif
constexpr bool kFastPath = YATT_A1_FASTPATH != 0;

// A1's ring waits: 0 = spin, 1 = the producer sleeps (suspend-time hint),
// 2 = producer and consumers sleep.  The producer's spin on free slots is
// ~11% of A1's issued instructions (ncu), yet spinning measured fastest in
// the sustained bench step on a power-capped box (10.16 / 10.10 / 10.08 M
// tok/s for 0 / 1 / 2, same box, two runs each): the wake-up latency of a
// sleeping waiter costs more than the issue slots the spin takes.  (The
// fused loss + gradient kernel, issue-bound, gains from sleeping waits.)
#ifndef YATT_A1_SLEEP
#define YATT_A1_SLEEP 0
#endif
__device__ __forceinline__ void a1_producer_wait(uint64_t* bar, uint32_t parity) {
  if (YATT_A1_SLEEP >= 1) mbar_sleep_wait(bar, parity);
  else mbar_wait(bar, parity);
}
__device__ __forceinline__ void a1_consumer_wait(uint64_t* bar, uint32_t parity) {
  if (YATT_A1_SLEEP >= 2) mbar_sleep_wait(bar, parity);
  else mbar_wait(bar, parity);
}
constexpr uint32_t kFixupSentinel = 0x7fc0fadeu;  // quiet NaN payload: "recompute me"
constexpr uint32_t kNegInf2 = 0xFF80FF80u;        // two bf16 -inf

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

// fp64 epilogue of one row from its combined partial and target logits.
__device__ __forceinline__ void emit_row(const A1Params& p, int64_t row, const RowPartial& q,
                                         double xy, double zy) {
  const double l2s = log2(double(q.s));
  const double l2q = log2(double(q.sq));
  const double logp = xy - kLn2 * (double(q.mp) + l2s);
  const double rlogp = zy - kLn2 * (double(q.mq) + l2q);
  // lse_q - lse_p without cancelling two large numbers.
  const double dlse = kLn2 * ((double(q.mq) - double(q.mp)) + log2(double(q.sq) / double(q.s)));
  p.logp[row] = float(logp);
  if (p.ref_logp) p.ref_logp[row] = float(rlogp);
  if (p.ent) p.ent[row] = float(kLn2 * (l2s - double(q.w) / double(q.s)));
  if (p.kl) {
    const double delta = (zy - xy) - dlse;  // ref_logp - logp
    double kl;
    switch (p.kl_mode) {
      case YATT_KL_K1: kl = -delta; break;
      case YATT_KL_K2: kl = 0.5 * delta * delta; break;
      case YATT_KL_K3: kl = expm1(delta) - delta; break;
      default: kl = double(q.u) / double(q.s) + dlse; break;
    }
    p.kl[row] = float(kl);
  }
}

// kEdges: V % 8 != 0 — rows are staged as 16-byte-aligned supersets and the
// edge vectors masked; false compiles the plain V % 8 == 0 kernel.
template <bool kFull, bool kEdges>
__global__ void __launch_bounds__(kThreads, kMinBlocks) token_stats_kernel(const A1Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem);
  SmemTail* tail = reinterpret_cast<SmemTail*>(smem + kRingBytes);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t V = p.V;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        if (p.mask != nullptr && p.mask[row] == 0) continue;
        // stage the row's 16-byte-aligned superset: h elements before it
        // (V % 8 != 0 only) and up to 7 after; consumers mask the edges
        const int h = kEdges ? int((row * V) & 7) : 0;
        const int64_t S = kEdges ? ((h + V + 7) & ~int64_t(7)) : V;
        const int ntiles_r = int((S + kTile - 1) / kTile);
        const uint16_t* gp = p.pol + row * V - h;
        const uint16_t* gq = p.ref + row * V - h;
        for (int t = 0; t < ntiles_r; ++t) {
          const int64_t e0 = int64_t(t) * kTile;
          const uint32_t n = uint32_t(min64(kTile, S - e0));
          a1_producer_wait(&tail->empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&tail->full[stage], 4u * n);
          uint16_t* dst = ring + size_t(stage) * 2 * kTile;
          bulk_g2s(dst, gp + e0, 2u * n, &tail->full[stage], pol);
          bulk_g2s(dst + kTile, gq + e0, 2u * n, &tail->full[stage], pol);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int tid = threadIdx.x;  // 0..kConsumers-1
  int stage = 0;
  uint32_t phase = 0;
  int iter = 0;
  // the next row's target prefetched a row ahead (the full KL, 8 more
  // accumulators live, loads it at the row start instead: no spills)
  int64_t next_row = blockIdx.x;
  int32_t y_next = !kFull && next_row < p.rows ? __ldg(p.tgt + next_row) : 0;
  Acc<kFull> acc;

  for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
    const int32_t y = (!kFull && row == next_row) ? y_next : __ldg(p.tgt + row);
    if (!kFull) {
      next_row = row + gridDim.x;
      if (next_row < p.rows) y_next = __ldg(p.tgt + next_row);
    }
    if (p.mask != nullptr && p.mask[row] == 0) {
      if (tid == 0) {
        p.logp[row] = 0.f;
        if (p.ref_logp) p.ref_logp[row] = 0.f;
        if (p.ent) p.ent[row] = 0.f;
        if (p.kl) p.kl[row] = 0.f;
      }
      continue;
    }
    const int par = iter & 1;
    const int h = kEdges ? int((row * V) & 7) : 0;  // staged row starts h elements early
    const int S = kEdges ? ((h + int(V) + 7) & ~7) : int(V);  // 32-bit: V < 2^31 - 15
    const int ntiles_r = (S + kTile - 1) / kTile;
    const int ty = (y + h) / kTile;    // tile holding the target logit
    const int yin = (y + h) - ty * kTile;
    acc.reset();

    for (int t = 0; t < ntiles_r; ++t) {
      const int e0 = t * kTile;
      const int nvec = min(kTile, S - e0) >> 3;
      const uint16_t* sp = ring + size_t(stage) * 2 * kTile;
      const uint16_t* sq = sp + kTile;
      a1_consumer_wait(&tail->full[stage], phase);
      if (t == ty && tid == 0 && y >= 0 && y < V) {  // target logits from the staged tile
        tail->tgt[par][0] = __uint_as_float(uint32_t(sp[yin]) << 16);
        tail->tgt[par][1] = __uint_as_float(uint32_t(sq[yin]) << 16);
      }
      // Whole tiles take an unpredicated path; a partial tile the same
      // unrolled code with vectors past the row end read as -inf (2^-inf = 0
      // in every sum, also after the floor).  (One shared predicated path
      // cost 26 -inf register fills + predicate logic per warp-tile, ~8% of
      // the tile's instructions.)
      auto tile = [&](auto whole_tag) {
        constexpr bool kWhole = decltype(whole_tag)::value;
        uint4 P[kVecPerThread], Q[kVecPerThread];
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i) {
          const int v = tid + i * kConsumers;
          const bool in = kWhole || v < nvec;
          P[i] = in ? lds128(sp + v * 8) : make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
          Q[i] = in ? lds128(sq + v * 8) : make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
          if (kEdges) {  // staged elements outside the row read as -inf
            const int j0 = e0 + v * 8 - h;  // row index of element 0
            if (in && (j0 < 0 || j0 + 8 > int(V))) {
              const int lo = max(0, -j0), hi = min(8, int(V) - j0);
              P[i] = keep_range(P[i], lo, hi);
              Q[i] = keep_range(Q[i], lo, hi);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i) {
          P[i] = floor_policy(P[i]);
          if (kFull) Q[i] = floor_policy(Q[i]);  // x - z finite when both are -inf
        }
        // Fast path: the per-thread bases come from the row's first tile only;
        // later tiles skip the max check (fewer instructions = less power on
        // this power-capped kernel).  A row whose later logits exceed a
        // thread's base by > ~88 nats overflows to inf, is flagged in the
        // epilogue and recomputed by token_stats_fixup_kernel.
        if (!kFastPath || t == 0) {
          uint32_t mpv = vmax4(P[0]), mqv = vmax4(Q[0]);
#pragma unroll
          for (int i = 1; i < kVecPerThread; ++i) {
            mpv = bmax2(mpv, vmax4(P[i]));
            mqv = bmax2(mqv, vmax4(Q[i]));
          }
          const float fmp = pair_max(mpv), fmq = pair_max(mqv);
          if (fmp > acc.thr_p) acc.rebase_p(fmp);
          if (fmq > acc.thr_q) acc.rebase_q(fmq);
        }
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i) acc.step(P[i], Q[i]);
      };
      if (nvec == kVecPerTile)
        tile(std::true_type{});
      else
        tile(std::false_type{});
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->empty[stage]);
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1u;
      }
    }

    // ---- row reduction: thread -> warp -> CTA ----
    RowPartial r;
    r.mp = acc.mp;
    r.mq = acc.mq;
    r.s = Acc<kFull>::total(acc.s);
    r.w = Acc<kFull>::total(acc.w);
    r.sq = Acc<kFull>::total(acc.sq);
    r.u = kFull ? Acc<kFull>::total(acc.u) : 0.f;
#if YATT_A1_NORMALIZE
    r = normalize(r);
#endif
    r = warp_combine<kFull>(r);
    if (lane == 0) tail->red[par][warp] = r;
    named_bar_sync(1, kConsumers);

    const int ew = iter & (kConsumerWarps - 1);  // rotating epilogue warp
    if (warp == ew) {
      RowPartial q = tail->red[par][lane & (kConsumerWarps - 1)];
#pragma unroll
      for (int off = kConsumerWarps / 2; off > 0; off >>= 1) q = combine(q, shfl_partial(q, off));
      if (lane == 0) {
        if (kFastPath && !partial_finite<kFull>(q)) {
          p.logp[row] = __uint_as_float(kFixupSentinel);  // token_stats_fixup_kernel redoes it
        } else {
          // a target outside [0, V) is a caller error: NaN log-probs / KL
          // (entropy stays valid), never an out-of-row access
          const bool yok = y >= 0 && y < V;
          const float nan = __uint_as_float(0x7fc00000u);
          emit_row(p, row, q, yok ? tail->tgt[par][0] : nan, yok ? tail->tgt[par][1] : nan);
        }
      }
    }
    ++iter;
  }
}

// 8 bf16 from an arbitrarily aligned row, -inf past the end (contributes 0).
__device__ __forceinline__ uint4 load8_any(const uint16_t* row, int64_t e0, int64_t V) {
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t lo = e0 + 2 * k < V ? uint32_t(__ldg(row + e0 + 2 * k)) : 0xFF80u;
    const uint32_t hi = e0 + 2 * k + 1 < V ? uint32_t(__ldg(row + e0 + 2 * k + 1)) : 0xFF80u;
    w[k] = lo | (hi << 16);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Robust per-row path, one CTA per row, per-vector rebase checks, global
// loads.  kGeneric = false: recompute the rows the fast path flagged
// (launched after every token_stats_kernel; with none flagged it only reads
// logp, 4 B/row).  kGeneric = true: every row, for vocabularies or tensors
// the TMA path cannot take (V % 8 != 0 or unaligned), with scalar loads.
template <bool kFull, bool kGeneric>
__global__ void __launch_bounds__(kConsumers) token_stats_fixup_kernel(const A1Params p) {
  __shared__ int64_t list[kConsumers];
  __shared__ int count;
  __shared__ RowPartial red[kConsumerWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t V = p.V;
  constexpr int kChunk = kGeneric ? 8 : kConsumers;  // rows examined per CTA iteration
  for (int64_t base = int64_t(blockIdx.x) * kChunk; base < p.rows;
       base += int64_t(gridDim.x) * kChunk) {
    if (tid == 0) count = 0;
    __syncthreads();
    const int64_t r = base + tid;
    if (tid < kChunk && r < p.rows) {
      if (kGeneric) {
        if (p.mask != nullptr && p.mask[r] == 0) {
          p.logp[r] = 0.f;
          if (p.ref_logp) p.ref_logp[r] = 0.f;
          if (p.ent) p.ent[r] = 0.f;
          if (p.kl) p.kl[r] = 0.f;
        } else {
          list[atomicAdd(&count, 1)] = r;
        }
      } else if (__float_as_uint(p.logp[r]) == kFixupSentinel) {
        list[atomicAdd(&count, 1)] = r;
      }
    }
    __syncthreads();
    const int n = count;
    for (int k = 0; k < n; ++k) {
      const int64_t row = list[k];
      Acc<kFull> acc;
      acc.reset();
      const uint16_t* rp = p.pol + row * V;
      const uint16_t* rq = p.ref + row * V;
      // rows of a V % 8 != 0 tensor are not 16-byte aligned (and a row's last
      // vector would run into the next row): element loads, masked at V
      const bool scalar = kGeneric || (V & 7) != 0;
      for (int64_t v = tid; v < (V + 7) / 8; v += kConsumers) {
        const uint4 P0 = scalar ? load8_any(rp, v * 8, V) : __ldg(reinterpret_cast<const uint4*>(rp) + v);
        const uint4 Q0 = scalar ? load8_any(rq, v * 8, V) : __ldg(reinterpret_cast<const uint4*>(rq) + v);
        const uint4 P = floor_policy(P0);
        const uint4 Q = kFull ? floor_policy(Q0) : Q0;
        const float fmp = pair_max(vmax4(P)), fmq = pair_max(vmax4(Q));
        if (fmp > acc.thr_p) acc.rebase_p(fmp);
        if (fmq > acc.thr_q) acc.rebase_q(fmq);
        acc.step(P, Q);
      }
      RowPartial q{acc.mp, Acc<kFull>::total(acc.s), Acc<kFull>::total(acc.w), acc.mq,
                   Acc<kFull>::total(acc.sq), kFull ? Acc<kFull>::total(acc.u) : 0.f};
      q = normalize(q);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) q = combine(q, shfl_partial(q, off));
      if (lane == 0) red[warp] = q;
      __syncthreads();
      if (warp == 0) {
        q = red[lane & (kConsumerWarps - 1)];
#pragma unroll
        for (int off = kConsumerWarps / 2; off > 0; off >>= 1) q = combine(q, shfl_partial(q, off));
        if (lane == 0) {
          const int32_t y = p.tgt[row];
          const bool yok = y >= 0 && y < V;  // else NaN log-probs / KL, no OOB read
          const float nan = __uint_as_float(0x7fc00000u);
          emit_row(p, row, q, yok ? __uint_as_float(uint32_t(p.pol[row * V + y]) << 16) : nan,
                   yok ? __uint_as_float(uint32_t(p.ref[row * V + y]) << 16) : nan);
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace

#ifndef YATT_FUSED_ONLY_TU  // token_stats_fused_{small,mid}.cu compile only the fused kernel
#ifdef YATT_A1_SMALL_TU
#define YATT_A1_RING token_stats_ring_small
#else
#define YATT_A1_RING token_stats_ring_large
#endif
// The TMA-ring path with this translation unit's ring shape (16-B-aligned
// tensors; with V % 8 != 0 the caller has peeled off the last row).
int YATT_A1_RING(const A1Params& p, cudaStream_t st) {
  const int32_t vocab = p.V, kl_mode = p.kl_mode;
  const int grid = int(min64(p.rows, int64_t(kMinBlocks) * num_sms()));
  {
    const bool edges = vocab % 8 != 0, full = kl_mode == YATT_KL_FULL;
    const void* k = edges ? (full ? reinterpret_cast<const void*>(token_stats_kernel<true, true>)
                                  : reinterpret_cast<const void*>(token_stats_kernel<false, true>))
                          : (full ? reinterpret_cast<const void*>(token_stats_kernel<true, false>)
                                  : reinterpret_cast<const void*>(token_stats_kernel<false, false>));
    const int rc_ = ensure_dynamic_smem(k, int(kSmemBytes));
    if (rc_) return rc_;
    if (edges) {
      if (full)
        token_stats_kernel<true, true><<<grid, kThreads, kSmemBytes, st>>>(p);
      else
        token_stats_kernel<false, true><<<grid, kThreads, kSmemBytes, st>>>(p);
    } else {
      if (full)
        token_stats_kernel<true, false><<<grid, kThreads, kSmemBytes, st>>>(p);
      else
        token_stats_kernel<false, false><<<grid, kThreads, kSmemBytes, st>>>(p);
    }
  }
  int rc = check_launch("token_stats_kernel");
  if (rc || !kFastPath) return rc;
  const int fgrid = int(min64(ceil_div(p.rows, kConsumers), int64_t(num_sms())));
  if (kl_mode == YATT_KL_FULL)
    token_stats_fixup_kernel<true, false><<<fgrid, kConsumers, 0, st>>>(p);
  else
    token_stats_fixup_kernel<false, false><<<fgrid, kConsumers, 0, st>>>(p);
  return check_launch("token_stats_fixup_kernel");
}

#endif  // !YATT_FUSED_ONLY_TU

#ifndef YATT_A1_SMALL_TU

// ======================================================================
// Training side (SURVEY.md §8f #1 fused with A1 and A4): the policy loss AND
// its gradient w.r.t. the policy logits in one kernel.  Per row the producer
// streams the policy logits twice through one policy-only ring: pass 1 with
// an L2 evict-normal policy (online log2 LSE + entropy, as A1, per-tile
// rebase so no fix-up pass is needed), pass 2 evict-first — the second read
// of the row is served from the 126 MB L2 (296 live rows x 304 KB at
// V=152,064).  Between the passes one warp forms the row's loss terms in
// fp64 (logp, H, the KL estimator against the stored ref_logp, the clipped
// surrogate's coefficient, grad_math.cuh) and hands them to all consumers
// through shared memory; pass 2 writes the bf16 gradient.  HBM bytes per
// row: 2V read + 2V written (+ ~20 B), vs 2V (A1 policy-only) + 4V (backward)
// for the two-kernel form.
// ======================================================================
struct FusedParams {
  const uint16_t* pol;
  const uint16_t* ref;    // reference logits (full-vocabulary KL only)
  const int32_t* tgt;
  const uint8_t* mask;
  const float* ref_logp;  // per-token reference log-prob (experience stage), may be null
  const float* old_logp;
  const float* adv;
  int64_t rows;
  int32_t V;
  int32_t kl_mode;  // K1 / K2 / K3
  yatt_loss_config cfg;
  double inv_norm;     // 1 / norm (token-mean: global valid tokens; seq modes: global sequences)
  const float* scale;  // seq-mean-token-mean: per-token 1 / (norm * valid tokens of its sequence)
  float* logp;
  float* ent;
  float* kl;
  uint16_t* grad;
};

namespace {

using gm::grad_vec;
using gm::pack_bf16x2;
using gm::store_grad;
using gm::target_grad;

// Shape: YATT_FUSED_CW consumer warps per CTA.  8: 2 CTAs/SM, 6 policy
// stages of 16 KB each (the small-vocabulary TU: 3 CTAs/SM, 4 stages); 16
// (the default for V > 60,000): one CTA per SM with 12 stages — the same
// warps and bytes in flight per SM but half the rows live between their two
// passes, so more of the second read hits L2: k3 3.76 vs 4.02 ms, full KL
// 6.07 vs 7.23 ms at 32,768 x 152,064 (r1_fused_grad_ncu_v1.md).
#ifndef YATT_FUSED_CW
#define YATT_FUSED_CW 16
#endif
constexpr int kFCW = YATT_FUSED_CW;
constexpr int kFC = kFCW * 32;
constexpr int kFThreads = kFC + 32;
constexpr int kFVpt = kVecPerTile / kFC;
constexpr int kFMinB = kFCW >= 16 ? 1 : kMinBlocks;
constexpr int kFStages = (kFCW >= 16 ? 4 : 2) * kStages;  // policy-only 16 KB stages
static_assert(kVecPerTile % kFC == 0 && (kFCW & (kFCW - 1)) == 0, "fused shape");
struct __align__(16) FusedTail {
  uint64_t full[kFStages];
  uint64_t empty[kFStages];
  RowPartial red[kFCW];
  float coef[8];  // g, h, f, lse_p, lse_q (log2 units), H, KL (gm::RowCoef order)
};
constexpr size_t kFusedSmem = size_t(kFStages) * kTile * sizeof(uint16_t) + sizeof(FusedTail);

__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}


// seq-mean-token-mean: per-token scale 1 / (norm * valid tokens of its
// sequence) — one CTA per sequence (grid-stride), tokens outside every
// sequence keep the zero the launcher wrote (zero gradient).
__global__ void __launch_bounds__(256) fused_seq_scale_kernel(const uint8_t* mask, const int64_t* cu,
                                                               int64_t nseq, double inv_norm,
                                                               float* scale) {
  __shared__ int red[8];
  for (int64_t sq = blockIdx.x; sq < nseq; sq += gridDim.x) {
    const int64_t b = cu[sq], e = cu[sq + 1];
    int cnt = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += 256) cnt += (mask == nullptr || mask[i]) ? 1 : 0;
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    int tot = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[k];
    const float sc = tot > 0 ? float(inv_norm / double(tot)) : 0.f;
    for (int64_t i = b + threadIdx.x; i < e; i += 256) scale[i] = sc;
    __syncthreads();
  }
}

// kFull: full-vocabulary KL — every stage holds the policy AND the reference
// tile (half the stages, the same bytes), pass 1 also accumulates lse_q and
// sum p (x - z), the epilogue forms KL = sum p (log p - log q) and the f
// coefficient, pass 2 uses the full gradient (grad_math.cuh).
template <bool kFull, bool kEdges>
__global__ void __launch_bounds__(kFThreads, kFMinB) policy_loss_grad_kernel(const FusedParams p) {
  constexpr int kPS = kFull ? 2 : 1;        // tiles per stage
  constexpr int kNS = kFStages / kPS;       // stages
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem);
  FusedTail* tail = reinterpret_cast<FusedTail*>(smem + size_t(kFStages) * kTile * sizeof(uint16_t));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t V = p.V;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], kFCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kFCW) {
    // ---------------- producer: every valid row twice ----------------
    if (lane == 0) {
      // pass 1 keeps the row in L2 for pass 2 (evict_last / applypriority
      // demotion measured no better: the rows' reuse distance, not priority,
      // sets the hit rate)
      const uint64_t keep = l2_evict_normal_policy(), drop = l2_evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        if (p.mask != nullptr && p.mask[row] == 0) continue;
        const int h = kEdges ? int((row * V) & 7) : 0;
        const int64_t S = kEdges ? ((h + V + 7) & ~int64_t(7)) : V;
        const int ntiles_r = int((S + kTile - 1) / kTile);
        const uint16_t* gp = p.pol + row * V - h;
        const uint16_t* gq = kFull ? p.ref + row * V - h : nullptr;
        for (int pass = 0; pass < 2; ++pass) {
          for (int t = 0; t < ntiles_r; ++t) {
            const int64_t e0 = int64_t(t) * kTile;
            const uint32_t n = uint32_t(min64(kTile, S - e0));
            mbar_wait(&tail->empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx(&tail->full[stage], 2u * n * kPS);
            uint16_t* dst = ring + size_t(stage) * kPS * kTile;
            const uint64_t pol = pass == 0 ? keep : drop;
            bulk_g2s(dst, gp + e0, 2u * n, &tail->full[stage], pol);
            if (kFull) bulk_g2s(dst + kTile, gq + e0, 2u * n, &tail->full[stage], pol);
            if (++stage == kNS) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int tid = threadIdx.x;
  int stage = 0;
  uint32_t phase = 0;
  Acc<kFull, kFull> acc;
  for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
    const int h = kEdges ? int((row * V) & 7) : 0;
    const int64_t S = kEdges ? ((h + V + 7) & ~int64_t(7)) : V;
    const int ntiles_r = int((S + kTile - 1) / kTile);
    uint16_t* gs = p.grad + row * V - h;  // staged coordinates
    if (p.mask != nullptr && p.mask[row] == 0) {
      if (tid == 0) {
        p.logp[row] = 0.f;
        if (p.ent) p.ent[row] = 0.f;
        if (p.kl) p.kl[row] = 0.f;
      }
      for (int64_t v = tid; v < S / 8; v += kFC)
        store_grad<kEdges>(gs, v * 8, make_uint4(0, 0, 0, 0), h, V);
      continue;
    }
    const int32_t y = __ldg(p.tgt + row);
    const int64_t ys = int64_t(y) + h;  // the target in staged coordinates
    const bool yok = y >= 0 && y < V;   // else NaN loss terms / gradient row, no OOB write
    float xy = yok ? 0.f : __uint_as_float(0x7fc00000u);  // the target logit (thread 0)
    // the row's per-token inputs, loaded now so the row-end epilogue (while
    // the other warps wait at the barrier) does not wait on global memory
    float r_old = 0.f, r_adv = 0.f, r_rl = 0.f, r_sc = 0.f;
    if (warp == 0 && lane < 2) {
      r_old = __ldg(p.old_logp + row);
      r_adv = __ldg(p.adv + row);
      r_rl = p.ref_logp ? __ldg(p.ref_logp + row) : 0.f;
      r_sc = p.scale ? __ldg(p.scale + row) : 0.f;
    }
    acc.reset();
    // ---- pass 1: online log2 LSE(s) + entropy (+ full-KL) sums ----
    for (int t = 0; t < ntiles_r; ++t) {
      const int64_t e0 = int64_t(t) * kTile;
      const int nvec = int(min64(kTile, S - e0) >> 3);
      const uint16_t* sp = ring + size_t(stage) * kPS * kTile;
      const uint16_t* sq = sp + kTile;
      mbar_wait(&tail->full[stage], phase);
      if (tid == 0 && yok && ys >= e0 && ys < e0 + kTile)
        xy = __uint_as_float(uint32_t(sp[ys - e0]) << 16);
      uint4 P[kFVpt], Q[kFVpt];
#pragma unroll
      for (int i = 0; i < kFVpt; ++i) {
        const int v = tid + i * kFC;
        const bool in = nvec == kVecPerTile || v < nvec;
        const uint4 ninf = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
        P[i] = in ? lds128(sp + v * 8) : ninf;
        Q[i] = kFull ? (in ? lds128(sq + v * 8) : ninf) : P[i];
        if (kEdges) {
          const int64_t j0 = e0 + int64_t(v) * 8 - h;
          if (in && (j0 < 0 || j0 + 8 > V)) {
            const int lo = int(max64(0, -j0)), hi = int(min64(8, V - j0));
            P[i] = keep_range(P[i], lo, hi);
            if (kFull) Q[i] = keep_range(Q[i], lo, hi);
          }
        }
        P[i] = floor_policy(P[i]);
        if (kFull) Q[i] = floor_policy(Q[i]);  // x - z finite when both are -inf
      }
      uint32_t mpv = vmax4(P[0]), mqv = kFull ? vmax4(Q[0]) : 0u;
#pragma unroll
      for (int i = 1; i < kFVpt; ++i) {
        mpv = bmax2(mpv, vmax4(P[i]));
        if (kFull) mqv = bmax2(mqv, vmax4(Q[i]));
      }
      const float fmp = pair_max(mpv);
      if (fmp > acc.thr_p) acc.rebase_p(fmp);
      if (kFull) {
        const float fmq = pair_max(mqv);
        if (fmq > acc.thr_q) acc.rebase_q(fmq);
      }
#pragma unroll
      for (int i = 0; i < kFVpt; ++i) acc.step(P[i], Q[i]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->empty[stage]);
      if (++stage == kNS) {
        stage = 0;
        phase ^= 1u;
      }
    }
    using A = Acc<kFull, kFull>;
    RowPartial r{acc.mp, A::total(acc.s), A::total(acc.w), kFull ? acc.mq : float(kMinitial),
                 kFull ? A::total(acc.sq) : 0.f, kFull ? A::total(acc.u) : 0.f};
    r = warp_combine<kFull>(r);
    if (lane == 0) tail->red[warp] = r;
    named_bar_sync(1, kFC);
    if (warp == 0) {
      RowPartial q = tail->red[lane & (kFCW - 1)];
#pragma unroll
      for (int off = kFCW / 2; off > 0; off >>= 1) q = combine(q, shfl_partial(q, off));
      // fp64 row epilogue: lane 0 forms logp / H (and the full KL), then lane
      // 0 takes the surrogate (exp of the ratio) while lane 1 takes the
      // per-token KL estimator (expm1) in parallel
      const double sc = p.scale ? double(r_sc) : p.inv_norm;
      double lp = 0.0;
      if (lane == 0) {
        const double l2s = log2(double(q.s));
        const double lse2 = double(q.mp) + l2s;
        lp = double(xy) - kLn2 * lse2;
        const double H = kLn2 * (l2s - double(q.w) / double(q.s));
        p.logp[row] = float(lp);
        if (p.ent) p.ent[row] = float(H);
        tail->coef[1] = float(sc * double(p.cfg.entropy_coef));
        tail->coef[3] = float(lse2);
        tail->coef[5] = float(H);
        if (kFull) {  // KL = sum p (log p - log q), without cancelling two lse
          const double dlse = kLn2 * ((double(q.mq) - double(q.mp)) +
                                      log2(double(q.sq) / double(q.s)));
          const double klf = double(q.u) / double(q.s) + dlse;
          if (p.kl) p.kl[row] = float(klf);
          tail->coef[2] = float(sc * double(p.cfg.kl_coef));
          tail->coef[4] = float(double(q.mq) + log2(double(q.sq)));
          tail->coef[6] = float(klf);
        } else {
          tail->coef[2] = tail->coef[4] = tail->coef[6] = 0.f;
        }
      }
      lp = __shfl_sync(0xffffffffu, lp, 0);
      double dkl = 0.0;
      if (!kFull && lane == 1) {  // the per-token KL estimator and its derivative
        const double delta = (p.ref_logp ? double(r_rl) : lp) - lp;
        double k;
        if (p.kl_mode == YATT_KL_K1) k = -delta, dkl = 1.0;
        else if (p.kl_mode == YATT_KL_K2) k = 0.5 * delta * delta, dkl = -delta;
        else {
          const double em1 = expm1(delta);
          k = em1 - delta;
          dkl = -em1;
        }
        if (p.kl) p.kl[row] = float(k);
      }
      dkl = __shfl_sync(0xffffffffu, dkl, 1);
      if (lane == 0) {
        const double g = gm::dloss_dlogp_pg(lp, double(r_old), double(r_adv), p.cfg) +
                         double(p.cfg.kl_coef) * dkl;
        tail->coef[0] = float(sc * g);
      }
    }
    named_bar_sync(1, kFC);
    const gm::RowCoef c{tail->coef[0], tail->coef[1], tail->coef[2], tail->coef[3],
                        tail->coef[4], tail->coef[5], tail->coef[6]};
    // ---- pass 2: the gradient (second read of the row, from L2) ----
    for (int t = 0; t < ntiles_r; ++t) {
      const int64_t e0 = int64_t(t) * kTile;
      const int nvec = int(min64(kTile, S - e0) >> 3);
      const uint16_t* sp = ring + size_t(stage) * kPS * kTile;
      const uint16_t* sq = sp + kTile;
      mbar_wait(&tail->full[stage], phase);
      if (nvec == kVecPerTile) {
        uint4 P[kFVpt], Q[kFVpt];
#pragma unroll
        for (int i = 0; i < kFVpt; ++i) {
          P[i] = floor_policy(lds128(sp + (tid + i * kFC) * 8));
          Q[i] = kFull ? floor_policy(lds128(sq + (tid + i * kFC) * 8)) : P[i];
        }
#pragma unroll
        for (int i = 0; i < kFVpt; ++i)
          store_grad<kEdges>(gs, e0 + (tid + i * kFC) * 8, grad_vec<kFull>(P[i], Q[i], c), h, V);
      } else {
        for (int v = tid; v < nvec; v += kFC) {
          const uint4 P = floor_policy(lds128(sp + v * 8));
          const uint4 Q = kFull ? floor_policy(lds128(sq + v * 8)) : P;
          store_grad<kEdges>(gs, e0 + v * 8, grad_vec<kFull>(P, Q, c), h, V);
        }
      }
      if (yok && ys >= e0 && ys < e0 + kTile && tid == ((ys - e0) >> 3) % kFC) {
        const float x = __uint_as_float(uint32_t(sp[ys - e0]) << 16);
        const float z = kFull ? __uint_as_float(uint32_t(sq[ys - e0]) << 16) : 0.f;
        gs[ys] = uint16_t(pack_bf16x2(target_grad<kFull>(x, z, c), 0.f) & 0xffffu);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->empty[stage]);
      if (++stage == kNS) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }
}

#if !defined(YATT_FUSED_ONLY_TU)
// ----------------------------------------------------------------------
// Large-vocabulary form of the fused loss + gradient: the kernel above with
// the row-end bubble and most of the instruction overhead removed.
//
// The kernel above is issue-bound, not HBM-bound (ncu, 8,192 x 152,064 k3:
// 19.8 thread instructions per logit for ~10 of arithmetic, issue 66%, DRAM
// 62%): every CTA stalls twice per row at named barriers around a one-warp
// fp64 epilogue, the consumers' per-tile bookkeeping is 64-bit, and the spin
// loops of idle warps take issue slots.  Here:
//   * a dedicated EPILOGUE warp owns the row end.  Consumers publish their
//     warp partials (double-buffered by row parity) and arrive on an
//     mbarrier; the epilogue warp combines them, derives the coefficients
//     pass 2 needs in fp32 (only a ratio within 1e-4 of a clip boundary
//     redoes the surrogate's branch from the fp64 log-prob) and releases the
//     consumers, then writes the fp64 per-token outputs off the critical path;
//   * pass 2 uses folded coefficients: t = c1 a + c0 (- f z), one FFMA2 per
//     pair instead of FMUL2 + FADD2 + FFMA2 (+ 3 for the full KL);
//   * 32-bit tile bookkeeping, full tiles unpredicated, and k3 stages of
//     16,384 logits (32 KB, 6 stages) so each warp's per-tile overhead covers
//     twice the work;
//   * every mbarrier wait carries a suspend-time hint, so waiting warps sleep
//     instead of spinning (the spin loops were ~9% of issued instructions).
// Pass order per row stays pass 1 -> pass 2 (pipelining pass 1 of the next
// row ahead, or splitting rows over a CTA cluster, was measured slower: the
// extra live rows overflow L2 / the cluster exchange couples the CTAs,
// profiles/r2_fused_pipe_v1.jsonl).  HBM bytes per row: 2V (4V full KL) read
// once, 2V written.
// ----------------------------------------------------------------------
// Kernel shapes.  Large vocabularies: one CTA per SM, 16 consumer warps and
// a 192 KB ring; small ones (V <= 60,000, short rows): 8 consumer warps, two
// CTAs per SM and a 96 KB ring each, so one CTA streams while the other is at
// its row end.
template <int kCW_, int kMinB_, int kRingBytes_, int kTileK3_, int kTileFull_>
struct PipeShape {
  static constexpr int kCW = kCW_;                // consumer warps
  static constexpr int kC = kCW * 32;             // consumer threads
  static constexpr int kThreads = kC + 64;        // + producer + epilogue warp
  static constexpr int kMinB = kMinB_;            // resident CTAs per SM
  static constexpr int kRing = kRingBytes_;       // smem ring bytes
  static constexpr int kTileK3 = kTileK3_;        // logits per stage (policy only)
  static constexpr int kTileFull = kTileFull_;    // logits per tensor per stage (pol + ref)
  static constexpr int kMaxStages = kRing / (2 * kTileK3) > kRing / (4 * kTileFull)
                                        ? kRing / (2 * kTileK3) : kRing / (4 * kTileFull);
};
using PipeLarge = PipeShape<16, 1, 196608, 16384, 8192>;
using PipeSmall = PipeShape<8, 2, 98304, 8192, 4096>;

template <class S>
struct __align__(16) PipeTail {
  uint64_t full[S::kMaxStages];
  uint64_t empty[S::kMaxStages];
  uint64_t pfull[2];  // consumer warps' partials published (count kCW)
  uint64_t cfull[2];  // row coefficients ready (count 1)
  RowPartial red[2][S::kCW];
  float2 xy[2];       // {target logit, valid}
  float coef[2][12];  // gm::RowCoef order, then the folded c1, c0, f
};
template <class S>
constexpr size_t pipe_smem() { return size_t(S::kRing) + sizeof(PipeTail<S>); }

// Gradient of 8 logits with the folded row coefficients:
//   a = x log2e - lse2, p = 2^a, t = c1 a + c0 (- f z), grad = p t
// (= p (h (log p + H) - g + f (log p - log q - KL)), grad_math.cuh).
template <bool kFull>
__device__ __forceinline__ uint4 grad_vec_folded(const uint4& P, const uint4& Q, float2 nl,
                                                 float2 c1, float2 c0, float2 nf) {
  const uint32_t pw[4] = {P.x, P.y, P.z, P.w};
  const uint32_t qw[4] = {Q.x, Q.y, Q.z, Q.w};
  uint32_t out[4];
  const float2 L2 = f2(kLog2e, kLog2e);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 a = __ffma2_rn(f2(bf16_lo(pw[k]), bf16_hi(pw[k])), L2, nl);
    const float2 e = ex2x2(a);
    float2 t = __ffma2_rn(c1, a, c0);
    if (kFull) t = __ffma2_rn(nf, f2(bf16_lo(qw[k]), bf16_hi(qw[k])), t);
    const float2 gr = __fmul2_rn(e, t);
    out[k] = pack_bf16x2(gr.x, gr.y);
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}

// Pass-2 tile order (kOrder): 0 forward, 1 reverse (the default).  In
// reverse the last tiles of pass 1 — the most recently read — are re-read
// first, so the tiles L2 still holds are taken before they age out: DRAM
// reads of the full-KL kernel 1.32x -> 1.23x the algorithmic bytes.  (Taking
// the ring-resident tail of pass 1 straight from shared memory cut DRAM
// reads further, to 1.13x, but ran slower — profiles/r2_fused_pipe_v6.jsonl.)
__device__ __forceinline__ int pass2_tile(int k, int ntiles, int order) {
  return order == 1 ? ntiles - 1 - k : k;
}

template <bool kFull, int kOrder, class S>
__global__ void __launch_bounds__(S::kThreads, S::kMinB) policy_loss_grad_pipe_kernel(
    const FusedParams p) {
  constexpr int kFCW = S::kCW, kFC = S::kC;
  constexpr int kPS = kFull ? 2 : 1;                          // tensors per stage
  constexpr int kPT = kFull ? S::kTileFull : S::kTileK3;      // logits per tensor per stage
  constexpr int kNS = S::kRing / (2 * kPS * kPT);             // stages
  constexpr int kPVec = kPT / 8;                              // 16-byte vectors per tensor tile
  constexpr int kPV = kPVec / kFC;                            // per consumer thread
  static_assert(kPVec % kFC == 0 && kNS >= 2 && kNS <= S::kMaxStages, "pipe shape");
  extern __shared__ __align__(128) uint8_t smem[];
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem);
  PipeTail<S>* tail = reinterpret_cast<PipeTail<S>*>(smem + S::kRing);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int V = p.V;
  const int ntiles = (V + kPT - 1) / kPT, nfull = V / kPT;
  const int last_nvec = (V - nfull * kPT) >> 3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], kFCW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tail->pfull[b], kFCW);
      mbar_init(&tail->cfull[b], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kFCW) {
    // ---------------- producer: every valid row twice ----------------
    if (lane == 0) {
      const uint64_t keep = l2_evict_normal_policy(), drop = l2_evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        if (p.mask != nullptr && p.mask[row] == 0) continue;
        const uint16_t* gp = p.pol + row * int64_t(V);
        const uint16_t* gq = kFull ? p.ref + row * int64_t(V) : nullptr;
        for (int pass = 0; pass < 2; ++pass) {
          for (int k = 0; k < ntiles; ++k) {
            const int t = pass == 0 ? k : pass2_tile(k, ntiles, kOrder);
            const int e0 = t * kPT;
            const uint32_t n = uint32_t(min(kPT, V - e0));
            // pass 1 keeps the row in L2 for pass 2 (evict-normal), pass 2 drops it
            const uint64_t pol = pass == 0 ? keep : drop;
            mbar_sleep_wait(&tail->empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx(&tail->full[stage], 2u * n * kPS);
            uint16_t* dst = ring + size_t(stage) * kPS * kPT;
            bulk_g2s(dst, gp + e0, 2u * n, &tail->full[stage], pol);
            if (kFull) bulk_g2s(dst + kPT, gq + e0, 2u * n, &tail->full[stage], pol);
            if (++stage == kNS) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == kFCW + 1) {
    // ---------------- epilogue warp: row partials -> coefficients ----------
    int j = 0;
    for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
      if (p.mask != nullptr && p.mask[row] == 0) continue;
      const int b = j & 1;
      // per-token inputs first: their latency hides under the wait
      float r_old = 0.f, r_adv = 0.f, r_rl = 0.f, r_sc = 0.f;
      if (lane < 2) {
        r_old = __ldg(p.old_logp + row);
        r_adv = __ldg(p.adv + row);
        r_rl = p.ref_logp ? __ldg(p.ref_logp + row) : 0.f;
        r_sc = p.scale ? __ldg(p.scale + row) : 0.f;
      }
      mbar_sleep_wait(&tail->pfull[b], uint32_t(j >> 1) & 1u);
      RowPartial q = tail->red[b][lane & (kFCW - 1)];
#pragma unroll
      for (int off = kFCW / 2; off > 0; off >>= 1) q = combine(q, shfl_partial(q, off));
      const float2 xyh = tail->xy[b];
      const float xy = xyh.y != 0.f ? xyh.x : __uint_as_float(0x7fc00000u);
      // (1) the coefficients pass 2 waits on, in fp32 (they scale a bf16
      // gradient); a ratio within 1e-4 of a clip boundary takes the branch
      // from the fp64 log-prob, so the clip decision is the fp64 one
      if (lane == 0) {
        const float sc = p.scale ? r_sc : float(p.inv_norm);
        const float l2s = log2f(q.s);
        const float lse2 = q.mp + l2s;
        const float lpf = xy - kLn2f * lse2;
        const float Hf = kLn2f * (l2s - q.w / q.s);
        const float h = sc * p.cfg.entropy_coef;
        float f = 0.f, lseq2 = 0.f, klf = 0.f;
        if (kFull) {
          f = sc * p.cfg.kl_coef;
          lseq2 = q.mq + log2f(q.sq);
          klf = q.u / q.s + kLn2f * ((q.mq - q.mp) + log2f(q.sq / q.s));
        }
        const float A = r_adv, ratio = expf(lpf - r_old);
        const float lo = 1.f - p.cfg.clip_low, hi = 1.f + p.cfg.clip_high;
        const float band = 1e-4f * ratio;
        bool near = fabsf(ratio - lo) <= band || fabsf(ratio - hi) <= band || !(ratio < 3e38f);
        float dpg;
        {
          const float pg1 = -A * ratio, pg2 = -A * fminf(fmaxf(ratio, lo), hi);
          const float pg = fmaxf(pg1, pg2);
          bool active = !(pg2 > pg1);
          if (p.cfg.clip_ratio_c > 1.f && A < 0.f) {
            const float bound = -A * p.cfg.clip_ratio_c;
            near = near || fabsf(pg - bound) <= 1e-4f * fabsf(bound);
            if (bound < pg) active = false;
          }
          dpg = active ? -A * ratio : 0.f;
        }
        if (near) {  // rare: the exact fp64 decision
          const double lp64 = double(xy) - kLn2 * (double(q.mp) + log2(double(q.s)));
          dpg = float(gm::dloss_dlogp_pg(lp64, double(r_old), double(A), p.cfg));
        }
        float dkl = 0.f;
        if (!kFull) {
          const float delta = (p.ref_logp ? r_rl : lpf) - lpf;
          dkl = p.kl_mode == YATT_KL_K1 ? 1.f : p.kl_mode == YATT_KL_K2 ? -delta : -expm1f(delta);
        }
        const float g = sc * (dpg + p.cfg.kl_coef * dkl);
        float* cf = tail->coef[b];
        cf[0] = g;
        cf[1] = h;
        cf[2] = f;
        cf[3] = lse2;
        cf[4] = lseq2;
        cf[5] = Hf;
        cf[6] = klf;
        cf[8] = (h + f) * kLn2f;
        cf[9] = fmaf(h, Hf, -g) + f * fmaf(kLn2f, lseq2, -klf);
        cf[10] = -f;
        mbar_arrive(&tail->cfull[b]);
      }
      // (2) the per-token outputs in fp64 (A1's numerics), off the critical
      // path: lane 0 logp / H (/ the full KL), lane 1 the KL estimator
      if (lane < 2) {
        const double l2s = log2(double(q.s));
        const double lp = double(xy) - kLn2 * (double(q.mp) + l2s);
        if (lane == 0) {
          p.logp[row] = float(lp);
          if (p.ent) p.ent[row] = float(kLn2 * (l2s - double(q.w) / double(q.s)));
          if (kFull && p.kl) {
            const double dlse = kLn2 * ((double(q.mq) - double(q.mp)) +
                                        log2(double(q.sq) / double(q.s)));
            p.kl[row] = float(double(q.u) / double(q.s) + dlse);
          }
        } else if (!kFull && p.kl) {
          const double delta = (p.ref_logp ? double(r_rl) : lp) - lp;
          double k;
          if (p.kl_mode == YATT_KL_K1) k = -delta;
          else if (p.kl_mode == YATT_KL_K2) k = 0.5 * delta * delta;
          else k = expm1(delta) - delta;
          p.kl[row] = float(k);
        }
      }
      __syncwarp();
      ++j;
    }
  } else {
    // ---------------- consumers ----------------
    const int tid = threadIdx.x;
    int stage = 0;
    uint32_t phase = 0;
    Acc<kFull, kFull> acc;
    const uint4 ninf = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
    int j = 0;
    for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
      uint16_t* gs = p.grad + row * int64_t(V);
      if (p.mask != nullptr && p.mask[row] == 0) {
        if (tid == 0) {
          p.logp[row] = 0.f;
          if (p.ent) p.ent[row] = 0.f;
          if (p.kl) p.kl[row] = 0.f;
        }
        for (int v = tid; v < V / 8; v += kFC) gm::stg_cs_128(gs + v * 8, make_uint4(0, 0, 0, 0));
        continue;
      }
      const int b = j & 1;
      const int32_t y = __ldg(p.tgt + row);
      const bool yok = y >= 0 && y < V;
      const int ty = yok ? y / kPT : -1, yin = yok ? y - ty * kPT : 0;
      float xy = 0.f;
      acc.reset();
      // ---- pass 1: online log2 LSE(s) + entropy (+ full-KL) sums ----
      for (int t = 0; t < ntiles; ++t) {
        const uint16_t* sp = ring + size_t(stage) * kPS * kPT;
        const uint16_t* sq = sp + kPT;
        const bool whole = t < nfull;
        mbar_sleep_wait(&tail->full[stage], phase);
        if (tid == 0 && t == ty) xy = __uint_as_float(uint32_t(sp[yin]) << 16);
        uint4 P[kPV], Q[kPV];
        if (whole) {
#pragma unroll
          for (int i = 0; i < kPV; ++i) {
            P[i] = floor_policy(lds128(sp + (tid + i * kFC) * 8));
            Q[i] = kFull ? floor_policy(lds128(sq + (tid + i * kFC) * 8)) : P[i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < kPV; ++i) {
            const int v = tid + i * kFC;
            P[i] = floor_policy(v < last_nvec ? lds128(sp + v * 8) : ninf);
            Q[i] = kFull ? floor_policy(v < last_nvec ? lds128(sq + v * 8) : ninf) : P[i];
          }
        }
        uint32_t mpv = vmax4(P[0]), mqv = kFull ? vmax4(Q[0]) : 0u;
#pragma unroll
        for (int i = 1; i < kPV; ++i) {
          mpv = bmax2(mpv, vmax4(P[i]));
          if (kFull) mqv = bmax2(mqv, vmax4(Q[i]));
        }
        const float fmp = pair_max(mpv);
        if (fmp > acc.thr_p) acc.rebase_p(fmp);
        if (kFull) {
          const float fmq = pair_max(mqv);
          if (fmq > acc.thr_q) acc.rebase_q(fmq);
        }
#pragma unroll
        for (int i = 0; i < kPV; ++i) acc.step(P[i], Q[i]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail->empty[stage]);
        if (++stage == kNS) {
          stage = 0;
          phase ^= 1u;
        }
      }
      using A = Acc<kFull, kFull>;
      RowPartial r{acc.mp, A::total(acc.s), A::total(acc.w), kFull ? acc.mq : float(kMinitial),
                   kFull ? A::total(acc.sq) : 0.f, kFull ? A::total(acc.u) : 0.f};
      r = warp_combine<kFull>(r);
      if (tid == 0) tail->xy[b] = make_float2(xy, yok ? 1.f : 0.f);
      if (lane == 0) {
        tail->red[b][warp] = r;
        mbar_arrive(&tail->pfull[b]);  // release: the partial (and xy) before it
      }
      // ---- pass 2: the gradient (second read of the row, from L2) ----
      mbar_sleep_wait(&tail->cfull[b], uint32_t(j >> 1) & 1u);
      const float* cf = tail->coef[b];
      const float2 nl = f2(-cf[3], -cf[3]), c1 = f2(cf[8], cf[8]), c0 = f2(cf[9], cf[9]),
                   nf = f2(cf[10], cf[10]);
      for (int k = 0; k < ntiles; ++k) {
        const int t = pass2_tile(k, ntiles, kOrder);
        const int e0 = t * kPT;
        const uint16_t* sp = ring + size_t(stage) * kPS * kPT;
        const uint16_t* sq = sp + kPT;
        mbar_sleep_wait(&tail->full[stage], phase);
        if (t < nfull) {
          uint4 P[kPV], Q[kPV];
#pragma unroll
          for (int i = 0; i < kPV; ++i) {
            P[i] = floor_policy(lds128(sp + (tid + i * kFC) * 8));
            Q[i] = kFull ? floor_policy(lds128(sq + (tid + i * kFC) * 8)) : P[i];
          }
#pragma unroll
          for (int i = 0; i < kPV; ++i)
            gm::stg_cs_128(gs + e0 + (tid + i * kFC) * 8,
                           grad_vec_folded<kFull>(P[i], Q[i], nl, c1, c0, nf));
        } else {
          for (int v = tid; v < last_nvec; v += kFC) {
            const uint4 P = floor_policy(lds128(sp + v * 8));
            const uint4 Q = kFull ? floor_policy(lds128(sq + v * 8)) : P;
            gm::stg_cs_128(gs + e0 + v * 8, grad_vec_folded<kFull>(P, Q, nl, c1, c0, nf));
          }
        }
        if (t == ty && tid == (yin >> 3) % kFC) {  // the target element carries + g
          const gm::RowCoef c{cf[0], cf[1], cf[2], cf[3], cf[4], cf[5], cf[6]};
          const float x = __uint_as_float(uint32_t(sp[yin]) << 16);
          const float z = kFull ? __uint_as_float(uint32_t(sq[yin]) << 16) : 0.f;
          gs[y] = uint16_t(pack_bf16x2(target_grad<kFull>(x, z, c), 0.f) & 0xffffu);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tail->empty[stage]);
        if (++stage == kNS) {
          stage = 0;
          phase ^= 1u;
        }
      }
      ++j;
    }
  }
}
#endif  // !YATT_FUSED_ONLY_TU

}  // namespace

#if !defined(YATT_FUSED_ONLY_TU)
int policy_loss_grad_ring_large(const FusedParams& p, cudaStream_t st);

// The issue-lean kernel: PipeLarge for V > 60,000, PipeSmall below (the
// caller dispatches; YATT_FUSED_ORDER = pass-2 tile order, measurement only).
template <class S>
int policy_loss_grad_pipe(const FusedParams& p, cudaStream_t st) {
  const bool full = p.kl_mode == YATT_KL_FULL;
  const char* ord_env = std::getenv("YATT_FUSED_ORDER");  // measurement only
  const int order = ord_env ? std::atoi(ord_env) : 1;
  YATT_REQUIRE(order == 0 || order == 1, YATT_ERR_CONFIG, "YATT_FUSED_ORDER must be 0 or 1");
  const void* const kernels[2][2] = {
      {reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<false, 0, S>),
       reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<false, 1, S>)},
      {reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<true, 0, S>),
       reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<true, 1, S>)}};
  const void* k = kernels[full ? 1 : 0][order];
  const int rc = ensure_dynamic_smem(k, int(pipe_smem<S>()));
  if (rc) return rc;
  const int grid = int(min64(p.rows, int64_t(S::kMinB) * num_sms()));
  void* args[] = {const_cast<FusedParams*>(&p)};
  YATT_TRY_CUDA(cudaLaunchKernel(k, dim3(unsigned(grid)), dim3(S::kThreads), args,
                                 pipe_smem<S>(), st));
  return check_launch("policy_loss_grad_pipe_kernel");
}
#endif

#if defined(YATT_FUSED_SMALL_TU)
#define YATT_FUSED_RING policy_loss_grad_ring_small
#elif defined(YATT_FUSED_MID_TU)
#define YATT_FUSED_RING policy_loss_grad_ring_mid
#else
#define YATT_FUSED_RING policy_loss_grad_ring_large
#endif
// The fused kernel with this translation unit's shape (validated params).
int YATT_FUSED_RING(const FusedParams& p, cudaStream_t st) {
  const int grid = int(min64(p.rows, int64_t(kFMinB) * num_sms()));
#ifdef YATT_FUSED_SMALL_TU  // the full-KL form would spill at 3 CTAs/SM: the mid TU takes it
  YATT_REQUIRE(p.kl_mode != YATT_KL_FULL, YATT_ERR_CONFIG, "policy_loss_grad: internal dispatch");
  const bool full = false;
  const void* k = reinterpret_cast<const void*>(policy_loss_grad_kernel<false, false>);
#else
  const bool full = p.kl_mode == YATT_KL_FULL;
  const void* k = full ? reinterpret_cast<const void*>(policy_loss_grad_kernel<true, false>)
                       : reinterpret_cast<const void*>(policy_loss_grad_kernel<false, false>);
#endif
  const int rc_ = ensure_dynamic_smem(k, int(kFusedSmem));
  if (rc_) return rc_;
#ifndef YATT_FUSED_SMALL_TU
  if (full)
    policy_loss_grad_kernel<true, false><<<grid, kFThreads, kFusedSmem, st>>>(p);
  else
#endif
    policy_loss_grad_kernel<false, false><<<grid, kFThreads, kFusedSmem, st>>>(p);
  (void)full;
  return check_launch("policy_loss_grad_kernel");
}

#ifndef YATT_FUSED_ONLY_TU
int policy_loss_grad_ring_small(const FusedParams& p, cudaStream_t st);  // token_stats_fused_small.cu
int policy_loss_grad_ring_mid(const FusedParams& p, cudaStream_t st);    // token_stats_fused_mid.cu
int a1_small_vmax();

size_t policy_loss_grad_workspace_bytes(int64_t rows, int32_t agg_mode) {
  return agg_mode == 1 ? size_t(max64(rows, 0)) * sizeof(float) : 0;
}

int policy_loss_grad_launch(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                            const uint8_t* mask, const float* ref_logp, const float* old_logp,
                            const float* adv,
                            int64_t rows, int32_t vocab, const int64_t* cu, int64_t nseq,
                            const yatt_loss_config* cfg, int32_t kl_mode, double norm,
                            float* logp, float* ent, float* kl, uint16_t* grad, void* ws,
                            size_t ws_bytes, cudaStream_t st) {
  YATT_REQUIRE(cfg != nullptr, YATT_ERR_CONFIG, "policy_loss_grad: null config");
  YATT_REQUIRE(norm > 0.0, YATT_ERR_CONFIG, "policy_loss_grad: norm must be > 0");
  YATT_REQUIRE(cfg->agg_mode >= 0 && cfg->agg_mode <= 2, YATT_ERR_CONFIG,
               "policy_loss_grad: unknown agg_mode %d", cfg->agg_mode);
  float* scale = nullptr;
  if (cfg->agg_mode == 1 && rows > 0) {  // seq-mean-token-mean: per-token scale
    YATT_REQUIRE(cu != nullptr && nseq > 0, YATT_ERR_CONFIG,
                 "policy_loss_grad: seq-mean-token-mean needs cu_seqlens");
    YATT_REQUIRE(ws != nullptr && ws_bytes >= policy_loss_grad_workspace_bytes(rows, 1),
                 YATT_ERR_WORKSPACE, "policy_loss_grad: workspace too small (%zu < %zu)",
                 ws_bytes, policy_loss_grad_workspace_bytes(rows, 1));
    scale = static_cast<float*>(ws);
    YATT_TRY_CUDA(cudaMemsetAsync(scale, 0, size_t(rows) * sizeof(float), st));
    fused_seq_scale_kernel<<<unsigned(min64(nseq, int64_t(8) * num_sms())), 256, 0, st>>>(
        mask, cu, nseq, 1.0 / norm, scale);
    const int rc = check_launch("fused_seq_scale_kernel");
    if (rc) return rc;
  }
  const FusedParams p{pol, ref, tgt, mask, ref_logp, old_logp, adv, rows, vocab, kl_mode, *cfg,
                      1.0 / norm, scale, logp, ent, kl, grad};
  YATT_REQUIRE(p.V > 0 && p.rows >= 0, YATT_ERR_CONFIG, "policy_loss_grad: bad shape");
  YATT_REQUIRE(p.kl_mode >= YATT_KL_K1 && p.kl_mode <= YATT_KL_FULL, YATT_ERR_CONFIG,
               "policy_loss_grad: unknown kl_mode %d", p.kl_mode);
  YATT_REQUIRE(p.kl_mode != YATT_KL_FULL || p.ref != nullptr, YATT_ERR_CONFIG,
               "policy_loss_grad: the full-vocabulary KL needs the reference logits");
  if (p.rows == 0) return YATT_OK;
  YATT_REQUIRE(p.pol && p.tgt && p.old_logp && p.adv && p.logp && p.grad, YATT_ERR_CONFIG,
               "policy_loss_grad: null pointer");
  // V % 8 != 0: a row's aligned staging superset can end past the tensor on
  // the last row; the aligned-V contract keeps the fused path simple
  YATT_REQUIRE(p.V % 8 == 0, YATT_ERR_CONFIG,
               "policy_loss_grad: vocab must be a multiple of 8 (got %d)", p.V);
  // Shape by vocabulary (k3 / full-KL fraction of the HBM roofline,
  // profiles/r2_fused_pipe_v8/v9.jsonl): the small pipe shape (2 CTAs/SM)
  // vs the large one (1 CTA/SM) at V=65,536 0.933 vs 0.861 / 0.857 vs 0.806;
  // 81,920 0.906 vs 0.911 / 0.844 vs 0.850; 98,304 0.862 vs 0.947 / 0.802 vs
  // 0.870.  YATT_FUSED_PIPE (measurement only): 1 / 2 = the large / small
  // pipe shape at any vocabulary, 0 = the round-1 kernels (3 CTAs/SM of 8
  // warps for V <= 60,000, the full KL at 2; one 16-warp CTA/SM above).
  constexpr int kFusedSmallVmax = 73728;
  const char* env = std::getenv("YATT_FUSED_PIPE");
  const int pipe = env ? std::atoi(env) : -1;
  if (pipe == 0) {
    if (p.V > a1_small_vmax()) return policy_loss_grad_ring_large(p, st);
    return p.kl_mode == YATT_KL_FULL ? policy_loss_grad_ring_mid(p, st)
                                     : policy_loss_grad_ring_small(p, st);
  }
  if (pipe == 2 || (pipe != 1 && p.V <= kFusedSmallVmax))
    return policy_loss_grad_pipe<PipeSmall>(p, st);
  return policy_loss_grad_pipe<PipeLarge>(p, st);
}

int token_stats_ring_small(const A1Params& p, cudaStream_t st);  // token_stats_small.cu

// Vocabularies up to this take the small ring shape (4,096-element tiles x 4
// stages, 3 CTAs/SM); larger ones the 8,192 x 3, 2 CTAs/SM shape.  Measured
// (B200, k3, L2 flushed), large vs small shape: V=8,192 3.58 vs 3.92 TB/s,
// 32,000 5.76 vs 5.95, 50,264 5.76 vs 6.18, 65,536 6.50 vs 6.29, 100,000 6.50
// vs 6.34, 128,256 6.64 vs 6.42, 152,064 6.84 vs 6.64.  YATT_A1_SMALL_VMAX
// overrides (measurement only).
#ifndef YATT_A1_SMALL_VMAX
#define YATT_A1_SMALL_VMAX 60000
#endif
int a1_small_vmax() {
  static const int v = [] {
    const char* e = std::getenv("YATT_A1_SMALL_VMAX");
    return e ? std::atoi(e) : YATT_A1_SMALL_VMAX;
  }();
  return v;
}

int token_stats_launch(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                       const uint8_t* mask, int64_t rows, int32_t vocab, int32_t kl_mode,
                       float* logp, float* ref_logp, float* ent, float* kl, cudaStream_t st) {
  YATT_REQUIRE(vocab > 0, YATT_ERR_CONFIG, "token_stats: vocab must be positive (got %d)", vocab);
  YATT_REQUIRE(rows >= 0, YATT_ERR_CONFIG, "token_stats: rows must be >= 0");
  YATT_REQUIRE(kl_mode >= YATT_KL_K1 && kl_mode <= YATT_KL_FULL, YATT_ERR_CONFIG,
               "token_stats: unknown kl_mode %d", kl_mode);
  if (rows == 0) return YATT_OK;
  YATT_REQUIRE(logp != nullptr, YATT_ERR_CONFIG, "token_stats: logp output is required");
  YATT_REQUIRE(pol && ref && tgt, YATT_ERR_CONFIG, "token_stats: null input pointer");
  A1Params p{pol, ref, tgt, mask, rows, vocab, kl_mode, logp, ref_logp, ent, kl};
  // The TMA path needs 16-byte-aligned tensor bases; any vocab: each row is
  // staged as its aligned superset.  With V % 8 != 0 the last row's superset
  // could end past the tensor, so that one row takes the generic kernel.
  // (V < 8 with V % 8 != 0: the superset of rows before the last can end
  // past the tensor too — those tiny vocabularies take the generic kernel.)
  const bool tma_ok = (reinterpret_cast<uintptr_t>(pol) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(ref) & 15) == 0 &&
                      (vocab % 8 == 0 || (rows > 1 && vocab > 8));
  if (tma_ok && vocab % 8 != 0) {
    A1Params last = p;
    const int64_t off = (rows - 1) * int64_t(vocab);
    last.pol = pol + off;
    last.ref = ref + off;
    last.tgt = tgt + (rows - 1);
    last.mask = mask ? mask + (rows - 1) : nullptr;
    last.rows = 1;
    last.logp = logp + (rows - 1);
    last.ref_logp = ref_logp ? ref_logp + (rows - 1) : nullptr;
    last.ent = ent ? ent + (rows - 1) : nullptr;
    last.kl = kl ? kl + (rows - 1) : nullptr;
    if (kl_mode == YATT_KL_FULL)
      token_stats_fixup_kernel<true, true><<<1, kConsumers, 0, st>>>(last);
    else
      token_stats_fixup_kernel<false, true><<<1, kConsumers, 0, st>>>(last);
    const int rc = check_launch("token_stats_generic_kernel");
    if (rc) return rc;
    p.rows = rows - 1;
  }
  if (!tma_ok) {  // generic path: unaligned tensors, scalar loads
    const int ggrid = int(min64(ceil_div(rows, 8), int64_t(num_sms()) * 8));
    if (kl_mode == YATT_KL_FULL)
      token_stats_fixup_kernel<true, true><<<ggrid, kConsumers, 0, st>>>(p);
    else
      token_stats_fixup_kernel<false, true><<<ggrid, kConsumers, 0, st>>>(p);
    return check_launch("token_stats_generic_kernel");
  }
  return vocab <= a1_small_vmax() ? token_stats_ring_small(p, st) : token_stats_ring_large(p, st);
}
#endif  // !YATT_FUSED_ONLY_TU
#endif

}  // namespace yattb
