// grad_math.cuh — per-element gradient of the policy loss w.r.t. the policy
// logits, shared by logits_backward.cu (the standalone
// backward) and token_stats.cu (the fused loss + gradient kernel).
//   d loss / d x_j = p_j * (-g + h (log p_j + H) + f (log p_j - log q_j - KL))
//                    + g [j == target]
// with per-row coefficients g (surrogate + per-token KL estimator), h
// (entropy bonus), f (full-vocabulary KL) and the row's lse / H / KL.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace yattb {
namespace gm {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2f = 0.69314718055994530942f;

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void stg_cs_128(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

struct RowCoef {
  float g, h, f, lsep2, lseq2, H, KL;  // lse in log2 units (lse * log2e)
};

// grad for 8 elements (one 16-byte vector) of policy P (and ref Q if kFull).
template <bool kFull>
__device__ __forceinline__ uint4 grad_vec(const uint4& P, const uint4& Q, const RowCoef& c) {
  const uint32_t pw[4] = {P.x, P.y, P.z, P.w};
  const uint32_t qw[4] = {Q.x, Q.y, Q.z, Q.w};
  uint32_t out[4];
  const float2 L2 = f2(kLog2e, kLog2e), nl = f2(-c.lsep2, -c.lsep2);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 x = f2(bf16_lo(pw[k]), bf16_hi(pw[k]));
    const float2 a = __ffma2_rn(x, L2, nl);            // log2 p
    const float2 p = f2(ex2_approx(a.x), ex2_approx(a.y));
    const float2 lnp = __fmul2_rn(a, f2(kLn2f, kLn2f));  // log p
    // g * (-p) + h * p * (log p + H)
    float2 t = __ffma2_rn(f2(c.h, c.h), __fadd2_rn(lnp, f2(c.H, c.H)), f2(-c.g, -c.g));
    if (kFull) {
      const float2 z = f2(bf16_lo(qw[k]), bf16_hi(qw[k]));
      const float2 lnq = __fmul2_rn(__ffma2_rn(z, L2, f2(-c.lseq2, -c.lseq2)), f2(kLn2f, kLn2f));
      const float2 d = __fadd2_rn(__fadd2_rn(lnp, f2(-lnq.x, -lnq.y)), f2(-c.KL, -c.KL));
      t = __ffma2_rn(f2(c.f, c.f), d, t);
    }
    const float2 gr = __fmul2_rn(p, t);
    out[k] = pack_bf16x2(gr.x, gr.y);
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}

// Stores one gradient vector at staged index j (of a row staged from h
// elements before its start); with kEdges, a vector straddling the row's
// ends writes only its in-row elements (the neighbours own the rest).
template <bool kEdges>
__device__ __forceinline__ void store_grad(uint16_t* gs, int64_t j, uint4 g, int h, int64_t V) {
  if (!kEdges || (j >= h && j + 8 <= h + V)) {
    stg_cs_128(gs + j, g);
    return;
  }
  const uint32_t w[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int64_t idx = j + k;
    if (idx >= h && idx < h + V) gs[idx] = uint16_t((w[k >> 1] >> (16 * (k & 1))) & 0xffffu);
  }
}


// The target element's value: the vector store wrote p_y * t_y; the exact
// gradient adds + g (x: policy logit, z: reference logit for kFull).
template <bool kFull>
__device__ __forceinline__ float target_grad(float x, float z, const RowCoef& c) {
  const float a = fmaf(x, kLog2e, -c.lsep2);
  const float pp = ex2_approx(a);
  float val = pp * fmaf(c.h, a * kLn2f + c.H, -c.g) + c.g;
  if (kFull) {
    const float lnq = fmaf(z, kLog2e, -c.lseq2) * kLn2f;
    val = fmaf(c.f * pp, a * kLn2f - lnq - c.KL, val);
  }
  return val;
}

// d(token loss)/d(logp) of the clipped surrogate (+ dual clip) and, except
// for the full-vocabulary KL (its gradient is the f term), beta * d(kl)/d(logp)
// of the per-token estimator; fp64 so clip decisions match the loss kernel.
// The clipped surrogate's part alone: d pg / d logp = -A ratio where the
// unclipped branch is active, 0 where the clip (or the dual clip) binds.
__device__ __forceinline__ double dloss_dlogp_pg(double lp, double old, double A,
                                                 const yatt_loss_config& c) {
  const double ratio = exp(lp - old);
  const double pg1 = -A * ratio;
  const double pg2 = -A * fmin(fmax(ratio, 1.0 - double(c.clip_low)), 1.0 + double(c.clip_high));
  const double pg = fmax(pg1, pg2);
  bool active = !(pg2 > pg1);
  if (c.clip_ratio_c > 1.f && A < 0.0 && -A * double(c.clip_ratio_c) < pg) active = false;
  return active ? -A * ratio : 0.0;
}

__device__ __forceinline__ double dloss_dlogp(double lp, double old, double A, double rl,
                                              const yatt_loss_config& c, int32_t kl_mode) {
  const double dpg = dloss_dlogp_pg(lp, old, A, c);
  double dkl = 0.0;
  if (kl_mode == YATT_KL_K1) dkl = 1.0;
  else if (kl_mode == YATT_KL_K2) dkl = lp - rl;
  else if (kl_mode == YATT_KL_K3) dkl = -expm1(rl - lp);
  return dpg + double(c.kl_coef) * dkl;
}

}  // namespace gm
}  // namespace yattb
