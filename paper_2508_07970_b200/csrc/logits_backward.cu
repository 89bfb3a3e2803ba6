// logits_backward.cu — §8f next #1: the loss gradient w.r.t. the policy
// logits, the Stage-4 consumer of A1 (token_stats) and A4 (policy_loss).
// Replaces the Training-stage cost stand-in (proj/src/simcore.cpp:404-406,
// PAPER.md:66) for the first backward step of the actor.
//
// With p = softmax(x_t), H = entropy, y the target and per-token scalars
//   g = s_t * (dpg/dlogp + beta * dkl/dlogp)    (k1/k2/k3 KL)
//   h = s_t * entropy_coef                      (loss has -entropy_coef * H)
//   f = s_t * beta                              (FULL KL only)
//   s_t = mask_t / norm  (norm = global token count, or per-seq for seq-mean)
// the gradient row is
//   dL/dx_v = g (1[v=y] - p_v) + h p_v (log p_v + H) + f p_v (log p_v - log q_v - KL)
// dpg/dlogp = -A * ratio on the unclipped branch, 0 when the clipped (or dual
// clipped) branch is active; dkl/dlogp = 1 (k1), logp - ref_logp (k2),
// 1 - exp(ref_logp - logp) (k3).
//
// Kernel 1 (grad_coef): per token, fp64, gathers the target logits to rebuild
//   lse_p = x_y - logp and lse_q = z_y - ref_logp; writes 8 floats per token.
// Kernel 2 (logits_backward): persistent, the A1 streaming design — a producer
//   warp feeds a 3-stage shared-memory ring with cp.async.bulk (policy tile, +
//   reference tile for FULL), 8 consumer warps compute the row with packed
//   f32x2 math and MUFU ex2, convert to bf16x2 and store 16 B per thread.
// Bytes per valid row: 2V read + 2V written (+2V read for FULL) + 32 B coef.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"
#include "grad_math.cuh"

namespace yattb {
namespace {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;
#ifndef YATT_BWD_TILE
#define YATT_BWD_TILE 8192
#endif
#ifndef YATT_BWD_STAGES
#define YATT_BWD_STAGES 6  // policy-only (k1/k2/k3) ring; FULL stages both tensors: half
#endif
#ifndef YATT_BWD_MINB
#define YATT_BWD_MINB 2
#endif
constexpr int kTile = YATT_BWD_TILE;
constexpr int kMinBlocks = YATT_BWD_MINB;
// Ring depth: ~96 KB in flight per CTA either way (policy-only tiles are half
// the size, so twice the stages).
constexpr int kMaxStages = YATT_BWD_STAGES;
template <bool kFull>
constexpr int stages_of() {
  return kFull ? YATT_BWD_STAGES / 2 : YATT_BWD_STAGES;
}
constexpr int kVecPerTile = kTile / 8;
constexpr int kVecPerThread = kVecPerTile / kConsumers;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2f = 0.69314718055994530942f;
constexpr int kCoef = 8;  // g, h, f, lse_p, lse_q, H, KL, pad

struct GradParams {
  const uint16_t* pol;
  const uint16_t* ref;
  const int32_t* tgt;
  const uint8_t* mask;
  const float* coef;
  int64_t rows;
  int32_t V;
  uint16_t* grad;
};

using gm::f2;
using gm::grad_vec;
using gm::pack_bf16x2;
using gm::RowCoef;
using gm::store_grad;
using gm::target_grad;

struct __align__(16) BwdTail {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
};

// kEdges: V % 8 != 0 — rows staged as 16-byte-aligned supersets (as in A1);
// the gradient tensor has the same layout, so interior vectors stay aligned.
template <bool kFull, bool kEdges>
__global__ void __launch_bounds__(kThreads, kMinBlocks) logits_backward_kernel(const GradParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kPerStage = kFull ? 2 : 1;
  constexpr int kStages = stages_of<kFull>();
  uint16_t* ring = reinterpret_cast<uint16_t*>(smem);
  BwdTail* tail = reinterpret_cast<BwdTail*>(smem + size_t(kStages) * kPerStage * kTile * 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        if (p.mask != nullptr && p.mask[row] == 0) continue;
        const int h = kEdges ? int((row * V) & 7) : 0;
        const int64_t S = kEdges ? ((h + V + 7) & ~int64_t(7)) : V;
        const int ntiles_r = int((S + kTile - 1) / kTile);
        for (int t = 0; t < ntiles_r; ++t) {
          const int64_t e0 = int64_t(t) * kTile;
          const uint32_t n = uint32_t(min64(kTile, S - e0));
          mbar_wait(&tail->empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&tail->full[stage], 2u * n * kPerStage);
          uint16_t* dst = ring + size_t(stage) * kPerStage * kTile;
          bulk_g2s(dst, p.pol + row * V - h + e0, 2u * n, &tail->full[stage], pol);
          if (kFull)
            bulk_g2s(dst + kTile, p.ref + row * V - h + e0, 2u * n, &tail->full[stage], pol);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    return;
  }

  const int tid = threadIdx.x;
  int stage = 0;
  uint32_t phase = 0;
  // per-row scalars, prefetched one row ahead (no load latency at row start)
  auto load_row = [&](int64_t r, float4& c0, float4& c1, int32_t& y) {
    if (r < p.rows) {
      const float4* cf = reinterpret_cast<const float4*>(p.coef + r * kCoef);
      c0 = __ldg(cf);
      c1 = __ldg(cf + 1);
      y = __ldg(p.tgt + r);
    }
  };
  float4 n0 = make_float4(0, 0, 0, 0), n1 = n0;
  int32_t ny = 0;
  load_row(blockIdx.x, n0, n1, ny);
  for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
    const float4 c0 = n0, c1 = n1;
    const int32_t y = ny;
    load_row(row + gridDim.x, n0, n1, ny);
    const int h = kEdges ? int((row * V) & 7) : 0;
    const int64_t S = kEdges ? ((h + V + 7) & ~int64_t(7)) : V;
    const int ntiles_r = int((S + kTile - 1) / kTile);
    uint16_t* gs = p.grad + row * V - h;  // staged coordinates
    if (p.mask != nullptr && p.mask[row] == 0) {
      for (int64_t v = tid; v < S / 8; v += kConsumers)
        store_grad<kEdges>(gs, v * 8, make_uint4(0, 0, 0, 0), h, V);
      continue;
    }
    const RowCoef c{c0.x, c0.y, c0.z, c0.w * kLog2e, c1.x * kLog2e, c1.y, c1.z};
    const int64_t ys = int64_t(y) + h;  // the target in staged coordinates
    for (int t = 0; t < ntiles_r; ++t) {
      const int64_t e0 = int64_t(t) * kTile;
      const int nvec = int(min64(kTile, S - e0) >> 3);
      const uint16_t* sp = ring + size_t(stage) * kPerStage * kTile;
      const uint16_t* sq = sp + kTile;
      mbar_wait(&tail->full[stage], phase);
      if (nvec == kVecPerTile) {
        uint4 P[kVecPerThread], Q[kVecPerThread];
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i) {
          P[i] = lds128(sp + (tid + i * kConsumers) * 8);
          Q[i] = kFull ? lds128(sq + (tid + i * kConsumers) * 8) : P[i];
        }
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i)
          store_grad<kEdges>(gs, e0 + (tid + i * kConsumers) * 8, grad_vec<kFull>(P[i], Q[i], c), h,
                             V);
      } else {
        for (int v = tid; v < nvec; v += kConsumers) {
          const uint4 P = lds128(sp + v * 8);
          const uint4 Q = kFull ? lds128(sq + v * 8) : P;
          store_grad<kEdges>(gs, e0 + v * 8, grad_vec<kFull>(P, Q, c), h, V);
        }
      }
      // the target element gets + g: its owner rewrites those two bytes
      // (same thread, program order after the vector store)
      if (y >= 0 && y < V && ys >= e0 && ys < e0 + kTile && tid == ((ys - e0) >> 3) % kConsumers) {
        const float x = __uint_as_float(uint32_t(sp[ys - e0]) << 16);
        const float z = kFull ? __uint_as_float(uint32_t(sq[ys - e0]) << 16) : 0.f;
        gs[ys] = uint16_t(pack_bf16x2(target_grad<kFull>(x, z, c), 0.f) & 0xffffu);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail->empty[stage]);
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1u;
      }
    }
  }
}

__device__ __forceinline__ float bf16_at(const uint16_t* base, int64_t idx) {
  return __uint_as_float(uint32_t(base[idx]) << 16);
}

// Any vocab / any 2-byte alignment (V % 8 != 0 or an unaligned view): one CTA
// per row, element-wise 2-byte loads and stores — the same per-element formula
// as the tile kernel's target patch, so both paths round identically.
template <bool kFull>
__global__ void __launch_bounds__(256) logits_backward_generic_kernel(const GradParams p) {
  const int64_t V = p.V;
  for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
    uint16_t* grow = p.grad + row * V;
    if (p.mask != nullptr && p.mask[row] == 0) {
      for (int64_t v = threadIdx.x; v < V; v += blockDim.x) grow[v] = 0;
      continue;
    }
    const float* cf = p.coef + row * kCoef;
    const RowCoef c{cf[0], cf[1], cf[2], cf[3] * kLog2e, cf[4] * kLog2e, cf[5], cf[6]};
    const int32_t y = p.tgt[row];
    const uint16_t* xp = p.pol + row * V;
    const uint16_t* xq = kFull ? p.ref + row * V : nullptr;
    for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
      const float a = fmaf(bf16_at(xp, v), kLog2e, -c.lsep2);
      const float pp = ex2_approx(a);
      float val = pp * fmaf(c.h, a * kLn2f + c.H, -c.g);
      if (kFull) {
        const float lnq = fmaf(bf16_at(xq, v), kLog2e, -c.lseq2) * kLn2f;
        val = fmaf(c.f * pp, a * kLn2f - lnq - c.KL, val);
      }
      if (v == y) val += c.g;
      grow[v] = uint16_t(pack_bf16x2(val, 0.f) & 0xffffu);
    }
  }
}

__global__ void grad_coef_kernel(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                                 const float* logp, const float* ref_logp, const float* old_logp,
                                 const float* adv, const float* ent, const float* kl,
                                 const uint8_t* mask, int64_t n, int32_t V, const int64_t* cu,
                                 int64_t nseq, const yatt_loss_config c, int32_t kl_mode,
                                 double norm, float* coef) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  float* o = coef + t * kCoef;
  const bool valid = mask == nullptr || mask[t];
  double scale = valid ? 1.0 / norm : 0.0;
  if (valid && c.agg_mode == 1) {  // seq-mean-token-mean: also / valid tokens of the sequence
    int64_t lo = 0, hi = nseq;     // find s with cu[s] <= t < cu[s+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (cu[mid] <= t) lo = mid;
      else hi = mid;
    }
    scale /= double(coef[cu[lo] * kCoef + 7]);  // count left by seq_count_kernel
  }
  const double lp = logp[t];
  const double rl = ref_logp ? double(ref_logp[t]) : lp;
  const double beta = double(c.kl_coef);
  const int32_t y = tgt[t];
  // a target outside [0, V) (caller error): NaN coefficients -> a NaN
  // gradient row, never an out-of-row read
  const bool yok = y >= 0 && y < V;
  const double xy = yok ? double(bf16_at(pol, t * int64_t(V) + y)) : __longlong_as_double(0x7ff8000000000000ll);
  o[0] = float(scale * gm::dloss_dlogp(lp, old_logp[t], adv[t], rl, c, kl_mode));
  o[1] = float(scale * double(c.entropy_coef));
  o[2] = float(kl_mode == YATT_KL_FULL ? scale * beta : 0.0);
  o[3] = float(xy - lp);  // lse_p
  o[4] = (kl_mode == YATT_KL_FULL && ref && yok) ? float(double(bf16_at(ref, t * int64_t(V) + y)) - rl)
                                                 : 0.f;
  o[5] = ent ? ent[t] : 0.f;
  o[6] = kl ? kl[t] : 0.f;
  // o[7] is scratch: the valid-token count of the sequence at its first token
}

// Valid tokens per sequence -> coef[cu[s]*8 + 7] (seq-mean-token-mean only).
__global__ void seq_count_kernel(const uint8_t* mask, const int64_t* cu, int64_t nseq,
                                 float* coef) {
  for (int64_t s = blockIdx.x; s < nseq; s += gridDim.x) {
    const int64_t b = cu[s], e = cu[s + 1];
    int cnt = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) cnt += (mask == nullptr || mask[i]);
    cnt = warp_sum(cnt);
    __shared__ int red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0 && e > b) {
      int tot = 0;
      for (int k = 0; k < int(blockDim.x >> 5); ++k) tot += red[k];
      coef[b * kCoef + 7] = float(tot);
    }
    __syncthreads();
  }
}

}  // namespace

int grad_coef_launch(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                     const float* logp, const float* ref_logp, const float* old_logp,
                     const float* adv, const float* ent, const float* kl, const uint8_t* mask,
                     int64_t n, int32_t V, const int64_t* cu, int64_t nseq,
                     const yatt_loss_config* cfg, int32_t kl_mode, double norm, float* coef,
                     cudaStream_t st) {
  YATT_REQUIRE(cfg != nullptr, YATT_ERR_CONFIG, "grad_coef: null config");
  YATT_REQUIRE(cfg->agg_mode >= 0 && cfg->agg_mode <= 2, YATT_ERR_CONFIG, "unknown agg_mode");
  YATT_REQUIRE(kl_mode >= 0 && kl_mode <= 3, YATT_ERR_CONFIG, "unknown kl_mode %d", kl_mode);
  YATT_REQUIRE(norm > 0, YATT_ERR_CONFIG, "grad_coef: norm must be positive");
  YATT_REQUIRE(cfg->agg_mode != 1 || cu != nullptr, YATT_ERR_CONFIG,
               "seq-mean-token-mean needs cu_seqlens");
  YATT_REQUIRE(kl_mode != YATT_KL_FULL || (ref && ref_logp), YATT_ERR_CONFIG,
               "FULL KL gradient needs the reference logits and ref_logp");
  if (n <= 0) return YATT_OK;
  if (cfg->agg_mode == 1 && nseq > 0) {
    seq_count_kernel<<<unsigned(min64(nseq, int64_t(num_sms()) * 8)), 256, 0, st>>>(mask, cu, nseq,
                                                                                   coef);
    const int rc = check_launch("seq_count_kernel");
    if (rc) return rc;
  }
  grad_coef_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(
      pol, ref, tgt, logp, ref_logp, old_logp, adv, ent, kl, mask, n, V, cu, nseq, *cfg, kl_mode,
      norm, coef);
  return check_launch("grad_coef_kernel");
}

int logits_backward_launch(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                           const uint8_t* mask, int64_t rows, int32_t V, const float* coef,
                           int32_t full_kl, uint16_t* grad, cudaStream_t st) {
  YATT_REQUIRE(V > 0, YATT_ERR_CONFIG, "logits_backward: vocab must be positive");
  YATT_REQUIRE(rows >= 0, YATT_ERR_CONFIG, "logits_backward: rows must be >= 0");
  if (rows == 0) return YATT_OK;
  YATT_REQUIRE(pol && tgt && coef && grad && (!full_kl || ref), YATT_ERR_CONFIG,
               "logits_backward: null pointer");
  GradParams prm{pol, ref, tgt, mask, coef, rows, V, grad};
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool tma_ok = a16(pol) && a16(grad) && (!full_kl || a16(ref)) && (V % 8 == 0 || (rows > 1 && V > 8));  // V < 8: see token_stats_launch
  auto generic = [&](const GradParams& g) {
    const int gg = int(min64(g.rows, int64_t(8) * num_sms()));
    if (full_kl)
      logits_backward_generic_kernel<true><<<gg, 256, 0, st>>>(g);
    else
      logits_backward_generic_kernel<false><<<gg, 256, 0, st>>>(g);
    return check_launch("logits_backward_generic_kernel");
  };
  if (!tma_ok) return generic(prm);
  const bool edges = V % 8 != 0;
  if (edges) {  // the last row's aligned superset could end past the tensors
    const int64_t off = (rows - 1) * int64_t(V);
    GradParams last{pol + off, full_kl ? ref + off : nullptr, tgt + (rows - 1),
                    mask ? mask + (rows - 1) : nullptr, coef + (rows - 1) * kCoef, 1, V,
                    grad + off};
    const int rc = generic(last);
    if (rc) return rc;
    prm.rows = rows - 1;
  }
  const int grid = int(min64(prm.rows, int64_t(kMinBlocks) * num_sms()));
  if (full_kl) {
    constexpr size_t smem = size_t(stages_of<true>()) * 2 * kTile * 2 + sizeof(BwdTail);
    const void* k = edges ? reinterpret_cast<const void*>(logits_backward_kernel<true, true>)
                          : reinterpret_cast<const void*>(logits_backward_kernel<true, false>);
    const int rc_ = ensure_dynamic_smem(k, int(smem));
    if (rc_) return rc_;
    if (edges)
      logits_backward_kernel<true, true><<<grid, kThreads, smem, st>>>(prm);
    else
      logits_backward_kernel<true, false><<<grid, kThreads, smem, st>>>(prm);
  } else {
    constexpr size_t smem = size_t(stages_of<false>()) * kTile * 2 + sizeof(BwdTail);
    const void* k = edges ? reinterpret_cast<const void*>(logits_backward_kernel<false, true>)
                          : reinterpret_cast<const void*>(logits_backward_kernel<false, false>);
    const int rc_ = ensure_dynamic_smem(k, int(smem));
    if (rc_) return rc_;
    if (edges)
      logits_backward_kernel<false, true><<<grid, kThreads, smem, st>>>(prm);
    else
      logits_backward_kernel<false, false><<<grid, kThreads, smem, st>>>(prm);
  }
  return check_launch("logits_backward_kernel");
}

}  // namespace yattb
