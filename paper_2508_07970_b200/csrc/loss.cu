// loss.cu — A4: fused clipped-surrogate + KL-penalty policy loss with masked
// token sums.  Replaces the Training-stage cost stand-in of the reference
// (proj/src/simcore.cpp:404-406) for the loss value itself.
//
// Per valid token t (the ratio / clip algebra in fp32 with the fp64 algebra
// for any token within 1e-4 of a clip bound, so every clip decision is the
// fp64 one; fp64 accumulation in a deterministic order; see Acc and add_vec):
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

// Per-thread accumulators.  Only the ratio/clip algebra is fp64 per token;
// loss_sum follows by linearity (sum L = sum pg + kl_coef sum kl -
// entropy_coef sum H), kl and H enter as fp32 sums of at most four tokens
// (one rounding per vector, relative 2^-23 of same-sign terms), counts are
// integers.
struct Acc {
  double pg = 0, ratio = 0, kl = 0, ent = 0;
  int32_t clip = 0, cnt = 0;
};
struct LossCfg {
  double lo, hi, cc;
  float flo, fhi, fcc;
  bool dual;
};
__device__ __forceinline__ LossCfg loss_cfg(const yatt_loss_config& c) {
  const double lo = 1.0 - double(c.clip_low), hi = 1.0 + double(c.clip_high);
  return LossCfg{lo, hi, double(c.clip_ratio_c), float(lo), float(hi), c.clip_ratio_c,
                 c.clip_ratio_c > 1.f};
}

// The ratio: fp32 expf (rel. error ~1e-7, incl. the fp32 difference), and the
// fp64 exp only where a decision could flip — within 1e-4 of a clip bound
// (or of the dual-clip bound), or an extreme value.  Every clip decision is
// then the fp64 one (the count is exact) and each summed term carries at most
// ~1e-7 relative error.  (Round 1 took the fp64 exp for every token.)
__device__ __forceinline__ double ratio_of(float logp, float old_logp, const LossCfg& c) {
  const float rf = expf(logp - old_logp);
  const float band = 1e-4f * rf;
  const bool near = fabsf(rf - c.flo) <= band || fabsf(rf - c.fhi) <= band ||
                    (c.dual && fabsf(rf - c.fcc) <= band) || !(rf < 3e38f) || !(rf > 1e-30f);
  return near ? exp(double(logp) - double(old_logp)) : double(rf);
}

__device__ __forceinline__ void pg_term(float logp, float old_logp, float A, const LossCfg& c,
                                        Acc& s) {
  const double ratio = ratio_of(logp, old_logp, c);
  const double a = double(A);
  const double pg1 = -a * ratio;
  const double pg2 = -a * fmin(fmax(ratio, c.lo), c.hi);
  double pg = fmax(pg1, pg2);
  s.clip += pg2 > pg1 ? 1 : 0;
  if (c.dual && a < 0.0) pg = fmin(pg, -a * c.cc);
  s.pg += pg;
  s.ratio += ratio;
  s.cnt += 1;
}

struct LossIn {
  const float *logp, *old_logp, *adv, *kl, *ent;
  const uint8_t* mask;
};

__device__ __forceinline__ float4 ldg4(const float* p, int64_t i) {
  return __ldg(reinterpret_cast<const float4*>(p + i));
}

// Token i (scalar path).
__device__ __forceinline__ void add_token(const LossIn& in, int64_t i, const LossCfg& c, Acc& s) {
  if (in.mask != nullptr && !in.mask[i]) return;
  pg_term(__ldg(in.logp + i), __ldg(in.old_logp + i), __ldg(in.adv + i), c, s);
  if (in.kl) s.kl += double(__ldg(in.kl + i));
  if (in.ent) s.ent += double(__ldg(in.ent + i));
}

// Four tokens [4j, 4j+4) from 16-byte loads (float inputs 16-B aligned, mask
// 4-B aligned).
struct Vec4 {
  float4 lp, olp, a;
  float k4, h4;  // masked kl / H sums of the four tokens, formed at load time so
  uint32_t m;    // two vectors in flight fit the 64-register cap without spills
};
__device__ __forceinline__ Vec4 load_vec(const LossIn& in, int64_t j) {
  Vec4 x;
  const int64_t i = 4 * j;
  x.lp = ldg4(in.logp, i);
  x.olp = ldg4(in.old_logp, i);
  x.a = ldg4(in.adv, i);
  x.m = in.mask ? __ldg(reinterpret_cast<const uint32_t*>(in.mask + i)) : 0x01010101u;
  const float4 kl = in.kl ? ldg4(in.kl, i) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 h = in.ent ? ldg4(in.ent, i) : make_float4(0.f, 0.f, 0.f, 0.f);
  // same order and rounding as the per-token loop it replaces: ((0 + t0) + t1) + ...
  x.k4 = 0.f;
  x.h4 = 0.f;
  if (x.m & 0xffu) x.k4 += kl.x, x.h4 += h.x;
  if ((x.m >> 8) & 0xffu) x.k4 += kl.y, x.h4 += h.y;
  if ((x.m >> 16) & 0xffu) x.k4 += kl.z, x.h4 += h.z;
  if (x.m >> 24) x.k4 += kl.w, x.h4 += h.w;
  return x;
}
// Four tokens of a vector in fp32, branch-free: clip decisions from the fp32
// ratio against the bounds (exact: a token within 1e-4 of a bound, or with an
// extreme ratio, takes the fp64 pg_term instead), pg = -A * (clipped ratio),
// the four pg / ratio values summed in fp32 (one rounding per add, like kl /
// H) and added to the fp64 accumulators once per vector.
__device__ __forceinline__ void add_vec(const Vec4& x, const LossCfg& c, Acc& s) {
  const float lp[4] = {x.lp.x, x.lp.y, x.lp.z, x.lp.w}, olp[4] = {x.olp.x, x.olp.y, x.olp.z, x.olp.w};
  const float a[4] = {x.a.x, x.a.y, x.a.z, x.a.w};
  float pg4 = 0.f, r4 = 0.f;
  int clip = 0, cnt = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool valid = ((x.m >> (8 * k)) & 0xffu) != 0;
    const float rf = __expf(lp[k] - olp[k]);  // ex2.approx: ~1e-6 relative for |d| <= 20
    const float band = 1e-4f * rf;
    const bool near = fabsf(rf - c.flo) <= band || fabsf(rf - c.fhi) <= band ||
                      (c.dual && fabsf(rf - c.fcc) <= band) || !(rf < 3e38f) || !(rf > 1e-30f);
    if (valid && near) {  // rare: the fp64 algebra decides
      pg_term(lp[k], olp[k], a[k], c, s);
      continue;
    }
    const bool clipped = (a[k] > 0.f && rf > c.fhi) || (a[k] < 0.f && rf < c.flo);
    float pg = -a[k] * (clipped ? fminf(fmaxf(rf, c.flo), c.fhi) : rf);
    if (c.dual && a[k] < 0.f) pg = fminf(pg, -a[k] * c.fcc);
    const bool use = valid && !near;
    pg4 += use ? pg : 0.f;
    r4 += use ? rf : 0.f;
    clip += (use && clipped) ? 1 : 0;
    cnt += use ? 1 : 0;
  }
  s.pg += double(pg4);
  s.ratio += double(r4);
  s.clip += clip;
  s.cnt += cnt;
  s.kl += double(x.k4);
  s.ent += double(x.h4);
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

// Writes the block's record: loss_sum from the linear combination unless the
// caller formed it per sequence (seq modes pass loss/seqs in v0/v7).
__device__ __forceinline__ void emit_part(const Acc& s, double v0, double v7,
                                          const yatt_loss_config& c, bool token_mode,
                                          double (*red)[kThreads / 32], double* part) {
  double v[kFields] = {v0, s.pg, s.kl, s.ent, double(s.clip), s.ratio, double(s.cnt), v7};
  block_sum(v, red);
  if (threadIdx.x == 0) {
    if (token_mode) v[0] = v[1] + double(c.kl_coef) * v[2] - double(c.entropy_coef) * v[3];
#pragma unroll
    for (int f = 0; f < kFields; ++f) part[kFields * blockIdx.x + f] = v[f];
  }
}

// agg_mode 0: contiguous ranges of 4-token vectors per block, two vectors in
// flight per thread; the n % 4 tail goes to the last block.
#ifndef YATT_LOSS_MINB  // 4 CTAs/SM (64 regs): token 57 us / seq 64 us vs 66 / 76 uncapped
#define YATT_LOSS_MINB 4
#endif
template <bool kVec>
__global__ void __launch_bounds__(kThreads, YATT_LOSS_MINB) loss_token_kernel(const LossIn in, int64_t n,
                                                              const yatt_loss_config cfg,
                                                              double* part) {
  __shared__ double red[kFields][kThreads / 32];
  const LossCfg c = loss_cfg(cfg);
  Acc s;
  if (kVec) {
    const int64_t nv = n >> 2;
    const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
    const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(nv, lo + per);
    int64_t j = lo + threadIdx.x;
    for (; j + kThreads < hi; j += 2 * kThreads) {
      const Vec4 x0 = load_vec(in, j), x1 = load_vec(in, j + kThreads);
      add_vec(x0, c, s);
      add_vec(x1, c, s);
    }
    if (j < hi) add_vec(load_vec(in, j), c, s);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < (n & 3)) add_token(in, 4 * nv + threadIdx.x, c, s);
  } else {
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(n, lo + per);
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) add_token(in, i, c, s);
  }
  emit_part(s, 0.0, 0.0, cfg, true, red, part);
}

// agg_mode 1/2: one CTA per sequence (grid-stride over sequences); the
// sequence's (pg, kl, H, count) are block-reduced to form its term, the other
// fields accumulate per thread.  Vector path: scalar head up to the first
// 4-aligned token, 16-byte body (two vectors in flight), scalar tail.
template <bool kVec>
#ifndef YATT_LOSS_SEQ_MINB  // the per-sequence kernel keeps more state live
#define YATT_LOSS_SEQ_MINB 3
#endif
__global__ void __launch_bounds__(kThreads, YATT_LOSS_SEQ_MINB) loss_seq_kernel(const LossIn in, const int64_t* cu,
                                                            int64_t nseq,
                                                            const yatt_loss_config cfg,
                                                            double* part) {
  __shared__ double red[kFields][kThreads / 32];
  __shared__ double sred[4][kThreads / 32];
  const LossCfg c = loss_cfg(cfg);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double beta = cfg.kl_coef, ec = cfg.entropy_coef;
  Acc tot;  // ratio / clip per thread; pg / kl / H / count from the block totals
  double loss = 0.0, seqs = 0.0;  // thread 0 only
  double t_pg = 0.0, t_kl = 0.0, t_ent = 0.0, t_cnt = 0.0;  // thread 0 only
  for (int64_t sq = blockIdx.x; sq < nseq; sq += gridDim.x) {
    const int64_t b = __ldg(cu + sq), e = __ldg(cu + sq + 1);
    Acc s;
    if (kVec) {
      const int64_t hb = min64(e, (b + 3) & ~int64_t(3));  // end of the scalar head
      const int64_t jb = hb >> 2, je = max64(jb, e >> 2);   // body vectors [jb, je)
      if (b + int64_t(threadIdx.x) < hb) add_token(in, b + threadIdx.x, c, s);
      int64_t j = jb + threadIdx.x;
      for (; j + kThreads < je; j += 2 * kThreads) {
        const Vec4 x0 = load_vec(in, j), x1 = load_vec(in, j + kThreads);
        add_vec(x0, c, s);
        add_vec(x1, c, s);
      }
      if (j < je) add_vec(load_vec(in, j), c, s);
      const int64_t tb = max64(hb, 4 * je);
      if (tb + int64_t(threadIdx.x) < e) add_token(in, tb + threadIdx.x, c, s);
    } else {
      for (int64_t i = b + threadIdx.x; i < e; i += kThreads) add_token(in, i, c, s);
    }
    double q[4] = {s.pg, s.kl, s.ent, double(s.cnt)};
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      q[f] = warp_sum(q[f]);
      if (lane == 0) sred[f][w] = q[f];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t[4] = {0, 0, 0, 0};
      for (int k = 0; k < kThreads / 32; ++k)
#pragma unroll
        for (int f = 0; f < 4; ++f) t[f] += sred[f][k];
      if (t[3] > 0) {
        const double Ls = t[0] + beta * t[1] - ec * t[2];
        loss += cfg.agg_mode == 1 ? Ls / t[3] : Ls;
        seqs += 1.0;
      }
      t_pg += t[0];
      t_kl += t[1];
      t_ent += t[2];
      t_cnt += t[3];
    }
    __syncthreads();
    tot.ratio += s.ratio;  // (fewer live doubles: no spills at the 64-register cap)
    tot.clip += s.clip;
  }
  if (threadIdx.x == 0) {
    tot.pg = t_pg;
    tot.kl = t_kl;
    tot.ent = t_ent;
    tot.cnt = int32_t(t_cnt);
  }
  emit_part(tot, loss, seqs, cfg, false, red, part);
}

}  // namespace


namespace {
constexpr int kMaxParts = 2048;
int token_parts() { return min(4 * num_sms(), kMaxParts); }
int seq_parts(int64_t nseq) { return int(max64(1, min64(nseq, int64_t(8) * num_sms()))); }
}  // namespace

size_t loss_workspace_bytes() { return size_t(kMaxParts) * kFields * sizeof(double); }

int policy_loss_parts_launch(const float* logp, const float* old_logp, const float* adv,
                             const float* kl, const float* ent, const uint8_t* mask, int64_t n,
                             const int64_t* cu, int64_t nseq, const yatt_loss_config* cfg,
                             void* ws, size_t ws_bytes, int* nparts, cudaStream_t st) {
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
  const int parts = cfg->agg_mode == 0 ? token_parts() : int(min64(seq_parts(nseq), kMaxParts));
  double* part = static_cast<double*>(ws);
  const LossIn in{logp, old_logp, adv, kl, ent, mask};
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool vec = a16(logp) && a16(old_logp) && a16(adv) && a16(kl) && a16(ent) &&
                   (reinterpret_cast<uintptr_t>(mask) & 3) == 0;
  if (cfg->agg_mode == 0) {
    if (vec)
      loss_token_kernel<true><<<parts, kThreads, 0, st>>>(in, n, *cfg, part);
    else
      loss_token_kernel<false><<<parts, kThreads, 0, st>>>(in, n, *cfg, part);
  } else {
    if (vec)
      loss_seq_kernel<true><<<parts, kThreads, 0, st>>>(in, cu, nseq, *cfg, part);
    else
      loss_seq_kernel<false><<<parts, kThreads, 0, st>>>(in, cu, nseq, *cfg, part);
  }
  *nparts = parts;
  return check_launch("policy_loss_kernel");
}

int policy_loss_launch(const float* logp, const float* old_logp, const float* adv,
                       const float* kl, const float* ent, const uint8_t* mask, int64_t n,
                       const int64_t* cu, int64_t nseq, const yatt_loss_config* cfg,
                       yatt_loss_sums* sums, void* ws, size_t ws_bytes, cudaStream_t st) {
  int parts = 0;
  const int rc = policy_loss_parts_launch(logp, old_logp, adv, kl, ent, mask, n, cu, nseq, cfg, ws,
                                          ws_bytes, &parts, st);
  if (rc) return rc;
  static_assert(sizeof(yatt_loss_sums) == kFields * sizeof(double), "yatt_loss_sums layout");
  reduce_parts_kernel<kFields><<<1, 256, 0, st>>>(static_cast<const double*>(ws), parts,
                                                   reinterpret_cast<double*>(sums));
  return check_launch("reduce_parts_kernel<8>");
}

double loss_finalize(const yatt_loss_sums* s, const yatt_loss_config* c) {
  if (s == nullptr || c == nullptr) return NAN;
  const double denom = c->agg_mode == 0 ? s->token_count : s->seq_count;
  return denom > 0 ? s->loss_sum / denom : 0.0;
}

}  // namespace yattb
