// policy_loss_grad.cu — SURVEY.md §8f #1 fused with A1 and A4: the
// training-side policy loss terms AND their gradient w.r.t. the policy
// logits in one kernel, from the policy logits alone.
//
// Replaces the Training-stage cost stand-in of the reference
// (proj/src/simcore.cpp:13-15, :404-406).  Per row the producer streams the
// policy logits twice through one TMA ring: pass 1 the online log2 LSE +
// entropy of A1 (online_lse.cuh; + the reference LSE and sum p (x - z) for
// the full-vocabulary KL), pass 2 the gradient (grad_math.cuh) — the second
// read served from the 126 MB L2.  HBM bytes per row: 2V read + 2V written
// (+ 2V read for the full KL), vs 2V (A1 policy-only) + 4V (backward) for the
// two-kernel form.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "grad_math.cuh"
#include "online_lse.cuh"

namespace yattb {

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

using gm::pack_bf16x2;
using gm::target_grad;

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

// ----------------------------------------------------------------------
// policy_loss_grad_pipe_kernel — one CTA runs rows start to end:
//   producer warp  one elected lane streams every valid row twice through a
//                  TMA bulk ring (pass 1 evict-normal so the row stays in L2,
//                  pass 2 evict-first and in REVERSE tile order: the most
//                  recently read tiles are re-read first, while L2 holds them)
//   consumers      pass 1: online log2 LSE + entropy (+ the full KL's
//                  reference LSE and sum p (x - z)), warp partials published
//                  (double-buffered by row parity) with an mbarrier arrive;
//                  pass 2: the gradient with FOLDED row coefficients,
//                  t = c1 a + c0 (- f z): one FFMA2 per pair
//   epilogue warp  combines the partials, derives pass 2's coefficients in
//                  fp32 (a ratio within 1e-4 of a clip boundary takes the
//                  surrogate's branch from the fp64 log-prob, so the clip
//                  decision is the fp64 one), releases the consumers, THEN
//                  writes the fp64 per-token outputs off the critical path.
// 32-bit tile bookkeeping, unpredicated whole tiles, and mbarrier waits with
// a suspend-time hint (spinning warps took ~9% of the issue slots of this
// issue-bound kernel).  Round 1's form (two named barriers per row around a
// one-warp fp64 epilogue, 19.8 instructions per logit) reached 0.82 (k3) /
// 0.75 (full KL) of the HBM roofline at V = 152,064; this one 0.969 / 0.874
// (profiles/r2_fused_grad_ncu.md).  Measured slower and dropped: pass 1 of
// the next row before pass 2 of this one (twice the live rows overflow L2),
// rows split over 2/4-CTA clusters with a DSMEM exchange of the partials
// (the exchange couples the CTAs), pass 2 taking the ring-resident tail of
// pass 1 from shared memory (profiles/r2_fused_pipe_v1..v6.jsonl).
//
// Shapes.  Large vocabularies: one CTA per SM, 16 consumer warps and a 192 KB
// ring; V <= 73,728 (short rows): 8 consumer warps, two CTAs per SM and a
// 96 KB ring each, so one CTA streams while the other is at its row end.
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

template <bool kFull, int kOrder, class S, int kLag>
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
      auto issue = [&](int64_t row, int pass) {
        const uint16_t* gp = p.pol + row * int64_t(V);
        const uint16_t* gq = kFull ? p.ref + row * int64_t(V) : nullptr;
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
      };
      // kLag = 1: pass 1 of row j before pass 2 of row j - 1 (the order the
      // consumers take them in)
      int64_t prev = -1;
      for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
        if (p.mask != nullptr && p.mask[row] == 0) continue;
        issue(row, 0);
        if (kLag == 0) {
          issue(row, 1);
        } else {
          if (prev >= 0) issue(prev, 1);
          prev = row;
        }
      }
      if (kLag != 0 && prev >= 0) issue(prev, 1);
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
    // ---- pass 2 of row `row` (the jr-th valid row): the gradient, second
    // read of the row from L2 ----
    auto pass2 = [&](int64_t row, int jr) {
      uint16_t* gs = p.grad + row * int64_t(V);
      const int32_t y = __ldg(p.tgt + row);
      const bool yok = y >= 0 && y < V;
      const int ty = yok ? y / kPT : -1, yin = yok ? y - ty * kPT : 0;
      mbar_sleep_wait(&tail->cfull[jr & 1], uint32_t(jr >> 1) & 1u);
      const float* cf = tail->coef[jr & 1];
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
    };
    int j = 0;
    int64_t prev = -1;
    for (int64_t row = blockIdx.x; row < p.rows; row += gridDim.x) {
      if (p.mask != nullptr && p.mask[row] == 0) {
        uint16_t* gs = p.grad + row * int64_t(V);
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
      if (kLag == 0) {
        pass2(row, j);
      } else {  // pass 1 of the next row first: the row end overlaps a whole pass
        if (prev >= 0) pass2(prev, j - 1);
        prev = row;
      }
      ++j;
    }
    if (kLag != 0 && prev >= 0) pass2(prev, j - 1);
  }
}
}  // namespace

// Launch with shape S (YATT_FUSED_ORDER = pass-2 tile order, measurement only).
template <class S, int kLag>
int policy_loss_grad_pipe_launch(const FusedParams& p, int order, cudaStream_t st) {
  const bool full = p.kl_mode == YATT_KL_FULL;
  const void* const kernels[2][2] = {
      {reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<false, 0, S, kLag>),
       reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<false, 1, S, kLag>)},
      {reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<true, 0, S, kLag>),
       reinterpret_cast<const void*>(policy_loss_grad_pipe_kernel<true, 1, S, kLag>)}};
  const void* k = kernels[full ? 1 : 0][order];
  const int rc = ensure_dynamic_smem(k, int(pipe_smem<S>()));
  if (rc) return rc;
  // YATT_FUSED_GRID: fewer CTAs than resident slots (measurement only)
  const char* ge = std::getenv("YATT_FUSED_GRID");
  const int64_t slots = int64_t(S::kMinB) * num_sms();
  const int grid = int(min64(p.rows, ge ? std::max<int64_t>(1, min64(slots, std::atoi(ge))) : slots));
  void* args[] = {const_cast<FusedParams*>(&p)};
  YATT_TRY_CUDA(cudaLaunchKernel(k, dim3(unsigned(grid)), dim3(S::kThreads), args,
                                 pipe_smem<S>(), st));
  return check_launch("policy_loss_grad_pipe_kernel");
}

// Launch with shape S; kLagDefault = whether pass 1 of the next row runs
// before pass 2 of this one (measurement only: YATT_FUSED_ORDER = pass-2
// tile order, YATT_FUSED_LAG = 0 / 1 overrides the lag).
template <class S, int kLagDefault>
int policy_loss_grad_pipe(const FusedParams& p, cudaStream_t st) {
  const char* ord_env = std::getenv("YATT_FUSED_ORDER");
  const int order = ord_env ? std::atoi(ord_env) : 1;
  YATT_REQUIRE(order == 0 || order == 1, YATT_ERR_CONFIG, "YATT_FUSED_ORDER must be 0 or 1");
  const char* lag_env = std::getenv("YATT_FUSED_LAG");
  const int lag = lag_env ? std::atoi(lag_env) : kLagDefault;
  return lag ? policy_loss_grad_pipe_launch<S, 1>(p, order, st)
             : policy_loss_grad_pipe_launch<S, 0>(p, order, st);
}

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
  if (p.rows == 0) return YATT_OK;  // (an empty tensor's data pointer may be null)
  YATT_REQUIRE(p.kl_mode != YATT_KL_FULL || p.ref != nullptr, YATT_ERR_CONFIG,
               "policy_loss_grad: the full-vocabulary KL needs the reference logits");
  YATT_REQUIRE(p.pol && p.tgt && p.old_logp && p.adv && p.logp && p.grad, YATT_ERR_CONFIG,
               "policy_loss_grad: null pointer");
  // V % 8 != 0: a row's aligned staging superset can end past the tensor on
  // the last row; the aligned-V contract keeps the fused path simple
  YATT_REQUIRE(p.V % 8 == 0, YATT_ERR_CONFIG,
               "policy_loss_grad: vocab must be a multiple of 8 (got %d)", p.V);
  // Shape by vocabulary, i.e. by how many rows can stay live in L2 between
  // their two passes (profiles/r2_fused_pipe_v11_lag.jsonl, fraction of the
  // HBM roofline, k3 / full KL):
  //   small shape (2 CTAs/SM) + lag (pass 1 of the next row before pass 2 of
  //     this one; 4 live rows per SM): k3 V=32,000 0.897 (no lag 0.830)
  //   large shape (1 CTA/SM) + lag (2 live rows per SM): k3 V=65,536 0.998
  //     (small 0.933, large 0.856); full KL V=32,000 0.780, 50,264 0.792,
  //     65,536 0.817 (small 0.770 / 0.769 / 0.819)
  //   large shape, no lag (1 live row per SM) above: k3 V=98,304 0.942 (with
  //     lag 0.796), 152,064 0.965 (0.691); full KL 98,304 0.863 (0.654)
  // YATT_FUSED_PIPE = 1 / 2 forces the large / small shape, YATT_FUSED_LAG
  // the lag (measurement only).
  constexpr int kSmallLagVmax = 36864, kLagVmax = 73728;
  const char* env = std::getenv("YATT_FUSED_PIPE");
  const int pipe = env ? std::atoi(env) : 0;
  const bool full = p.kl_mode == YATT_KL_FULL;
  if (pipe == 2 || (pipe == 0 && !full && p.V <= kSmallLagVmax))
    return policy_loss_grad_pipe<PipeSmall, 1>(p, st);
  if (p.V <= kLagVmax) return policy_loss_grad_pipe<PipeLarge, 1>(p, st);
  return policy_loss_grad_pipe<PipeLarge, 0>(p, st);
}

}  // namespace yattb
