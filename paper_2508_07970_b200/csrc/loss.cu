// loss.cu — A4: fused clipped-surrogate + KL-penalty policy loss with masked
// token sums.  Replaces the Training-stage cost stand-in of the reference
// (proj/src/simcore.cpp:404-406) for the loss value itself.
//
// Per valid token t (fp64 arithmetic, deterministic reduction order):
//   ratio = exp(logp - old_logp)
//   pg    = max(-A*ratio, -A*clip(ratio, 1-eps_lo, 1+eps_hi))     [clipped if 2nd > 1st]
//   dual clip (clip_ratio_c > 1, A < 0): pg = min(pg, -A*clip_ratio_c)
//   L     = pg + kl_coef*kl - entropy_coef*H
// Aggregation (yatt_loss_config.agg_mode):
//   0 token-mean          loss_sum = sum_t m L,              loss = loss_sum / token_count
//   1 seq-mean-token-mean loss_sum = sum_s (sum_t m L / n_s), loss = loss_sum / seq_count
//   2 seq-mean-token-sum  loss_sum = sum_s  sum_t m L,        loss = loss_sum / seq_count
// token_count / seq_count are all-reduced across ranks before the division
// (the only cross-rank traffic of the step).
// Bytes per token: logp, old_logp, adv, kl, entropy (4 B each) + mask (1 B).
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace yattb {
namespace {

constexpr int kThreads = 256;
constexpr int kFields = 8;  // yatt_loss_sums fields

struct TokenTerms {
  double L, pg, kl, ent, clipped, ratio;
};

__device__ __forceinline__ TokenTerms token_terms(float logp, float old_logp, float A, float kl,
                                                  float H, const yatt_loss_config& c) {
  TokenTerms t;
  const double ratio = exp(double(logp) - double(old_logp));
  const double a = double(A);
  const double pg1 = -a * ratio;
  const double lo = 1.0 - double(c.clip_low), hi = 1.0 + double(c.clip_high);
  const double pg2 = -a * fmin(fmax(ratio, lo), hi);
  double pg = fmax(pg1, pg2);
  t.clipped = pg2 > pg1 ? 1.0 : 0.0;
  if (c.clip_ratio_c > 1.f && a < 0.0) pg = fmin(pg, -a * double(c.clip_ratio_c));
  t.pg = pg;
  t.kl = double(kl);
  t.ent = double(H);
  t.L = pg + double(c.kl_coef) * t.kl - double(c.entropy_coef) * t.ent;
  t.ratio = ratio;
  return t;
}

// Block-wide sum of kFields doubles; result valid in thread 0.
__device__ __forceinline__ void block_sum(double (&v)[kFields], double (*red)[kThreads / 32]) {
#pragma unroll
  for (int f = 0; f < kFields; ++f) v[f] = warp_sum(v[f]);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int f = 0; f < kFields; ++f) red[f][w] = v[f];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < kFields; ++f) {
      double s = 0;
      for (int i = 0; i < kThreads / 32; ++i) s += red[f][i];
      v[f] = s;
    }
  }
}

// agg_mode 0: contiguous token ranges per block.
__global__ void __launch_bounds__(kThreads) loss_token_kernel(
    const float* logp, const float* old_logp, const float* adv, const float* kl,
    const float* ent, const uint8_t* mask, int64_t n, const yatt_loss_config c, double* part) {
  __shared__ double red[kFields][kThreads / 32];
  double v[kFields] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(n, lo + per);
  for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
    if (mask != nullptr && !mask[i]) continue;
    const TokenTerms t = token_terms(logp[i], old_logp[i], adv[i], kl ? kl[i] : 0.f,
                                     ent ? ent[i] : 0.f, c);
    v[0] += t.L;
    v[1] += t.pg;
    v[2] += t.kl;
    v[3] += t.ent;
    v[4] += t.clipped;
    v[5] += t.ratio;
    v[6] += 1.0;
  }
  block_sum(v, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < kFields; ++f) part[kFields * blockIdx.x + f] = v[f];
  }
}

// agg_mode 1/2: one warp per sequence; the sequence term is formed in-warp.
__global__ void __launch_bounds__(kThreads) loss_seq_kernel(
    const float* logp, const float* old_logp, const float* adv, const float* kl,
    const float* ent, const uint8_t* mask, const int64_t* cu, int64_t nseq,
    const yatt_loss_config c, double* part) {
  __shared__ double red[kFields][kThreads / 32];
  double v[kFields] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int lane = threadIdx.x & 31;
  const int64_t per = (nseq + gridDim.x - 1) / gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(nseq, lo + per);
  for (int64_t s = lo + (threadIdx.x >> 5); s < hi; s += kThreads / 32) {
    double sl = 0, cnt = 0;
    for (int64_t i = cu[s] + lane; i < cu[s + 1]; i += 32) {
      if (mask != nullptr && !mask[i]) continue;
      const TokenTerms t = token_terms(logp[i], old_logp[i], adv[i], kl ? kl[i] : 0.f,
                                       ent ? ent[i] : 0.f, c);
      sl += t.L;
      v[1] += t.pg;
      v[2] += t.kl;
      v[3] += t.ent;
      v[4] += t.clipped;
      v[5] += t.ratio;
      cnt += 1.0;
    }
    sl = warp_sum(sl);
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt > 0) {
      v[0] += c.agg_mode == 1 ? sl / cnt : sl;
      v[6] += cnt;
      v[7] += 1.0;
    }
  }
  block_sum(v, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < kFields; ++f) part[kFields * blockIdx.x + f] = v[f];
  }
}

__global__ void loss_final_kernel(const double* part, int nparts, int32_t agg_mode,
                                  yatt_loss_sums* out) {
  const int f = threadIdx.x;
  if (f >= kFields) return;
  double s = 0;
  for (int i = 0; i < nparts; ++i) s += part[kFields * i + f];
  double* o = reinterpret_cast<double*>(out);
  o[f] = s;
  (void)agg_mode;
}

int loss_parts() { return min(2 * num_sms(), 512); }

}  // namespace

size_t loss_workspace_bytes() { return size_t(512) * kFields * sizeof(double); }

int policy_loss_launch(const float* logp, const float* old_logp, const float* adv,
                       const float* kl, const float* ent, const uint8_t* mask, int64_t n,
                       const int64_t* cu, int64_t nseq, const yatt_loss_config* cfg,
                       yatt_loss_sums* sums, void* ws, size_t ws_bytes, cudaStream_t st) {
  YATT_REQUIRE(cfg != nullptr, YATT_ERR_CONFIG, "policy_loss: null config");
  YATT_REQUIRE(cfg->agg_mode >= 0 && cfg->agg_mode <= 2, YATT_ERR_CONFIG,
               "policy_loss: unknown agg_mode %d", cfg->agg_mode);
  YATT_REQUIRE(cfg->clip_low >= 0.f && cfg->clip_low < 1.f && cfg->clip_high >= 0.f,
               YATT_ERR_CONFIG, "policy_loss: clip range must satisfy 0 <= eps_low < 1, eps_high >= 0");
  YATT_REQUIRE(n >= 0 && nseq >= 0, YATT_ERR_CONFIG, "policy_loss: negative size");
  YATT_REQUIRE(cfg->agg_mode == 0 || cu != nullptr, YATT_ERR_CONFIG,
               "policy_loss: seq-mean modes need cu_seqlens");
  YATT_REQUIRE(ws_bytes >= loss_workspace_bytes() && ws != nullptr, YATT_ERR_WORKSPACE,
               "policy_loss: workspace too small (%zu < %zu)", ws_bytes, loss_workspace_bytes());
  const int parts = loss_parts();
  double* part = static_cast<double*>(ws);
  if (cfg->agg_mode == 0) {
    loss_token_kernel<<<parts, kThreads, 0, st>>>(logp, old_logp, adv, kl, ent, mask, n, *cfg,
                                                  part);
  } else {
    loss_seq_kernel<<<parts, kThreads, 0, st>>>(logp, old_logp, adv, kl, ent, mask, cu, nseq,
                                                *cfg, part);
  }
  int rc = check_launch("policy_loss_kernel");
  if (rc) return rc;
  loss_final_kernel<<<1, 32, 0, st>>>(part, parts, cfg->agg_mode, sums);
  return check_launch("loss_final_kernel");
}

double loss_finalize(const yatt_loss_sums* s, const yatt_loss_config* c) {
  if (s == nullptr || c == nullptr) return NAN;
  const double denom = c->agg_mode == 0 ? s->token_count : s->seq_count;
  return denom > 0 ? s->loss_sum / denom : 0.0;
}

}  // namespace yattb
