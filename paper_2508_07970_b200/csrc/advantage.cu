// advantage.cu — A2 GRPO group advantages and A3 PPO GAE (+ whitening).
//
// Both replace parts of the reference's Preparation stand-in
// (proj/src/simcore.cpp:395-398; "the critic computes values").
// Groups follow the reference's per-group unit: group = sample_id / G on
// GLOBAL sample ids (proj/src/workload.cpp:158-160, runner.cpp:158-160).
// All arithmetic is fp64 on the device (tiny byte counts; this keeps the
// results within an ulp of the fp64 oracle even where the scan reassociates).
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace yattb {
namespace {

// ---------------------------------------------------------------- GRPO ----
struct Moments {
  double n, mean, m2;
};

// Two-pass (mean, M2) over the local members of global group g.
__device__ __forceinline__ Moments local_group_moments(const float* r, int64_t n,
                                                       uint64_t first_id, int32_t G, uint64_t g) {
  const int64_t lo = max64(0, int64_t(g * uint64_t(G)) - int64_t(first_id));
  const int64_t hi = min64(n, int64_t((g + 1) * uint64_t(G)) - int64_t(first_id));
  Moments m{double(hi - lo), 0.0, 0.0};
  double sum = 0.0;
  for (int64_t i = lo; i < hi; ++i) sum += double(r[i]);
  m.mean = m.n > 0 ? sum / m.n : 0.0;
  for (int64_t i = lo; i < hi; ++i) {
    const double d = double(r[i]) - m.mean;
    m.m2 += d * d;
  }
  return m;
}

__global__ void grpo_moments_kernel(const float* r, int64_t n, uint64_t first_id, int32_t G,
                                    int64_t ngroups, double* out) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= ngroups) return;
  const uint64_t g = first_id / uint64_t(G) + uint64_t(k);
  const Moments m = local_group_moments(r, n, first_id, G, g);
  out[3 * k + 0] = m.n;
  out[3 * k + 1] = m.mean;
  out[3 * k + 2] = m.m2;
}

__global__ void grpo_adv_kernel(const float* r, int64_t n, uint64_t first_id, int32_t G,
                                float eps, int32_t norm_by_std, const double* moments,
                                float* adv) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t g = (first_id + uint64_t(i)) / uint64_t(G);
  Moments m;
  if (moments != nullptr) {
    const int64_t k = int64_t(g - first_id / uint64_t(G));
    m = Moments{moments[3 * k], moments[3 * k + 1], moments[3 * k + 2]};
  } else {
    m = local_group_moments(r, n, first_id, G, g);
  }
  double a = 0.0;
  if (m.n > 1.0) {
    const double centered = double(r[i]) - m.mean;
    if (norm_by_std) {
      const double sd = sqrt(m.m2 / (m.n - 1.0));
      a = centered / (sd + double(eps));
    } else {
      a = centered;
    }
  }
  adv[i] = float(a);
}

__global__ void broadcast_kernel(const float* vals, const int64_t* cu, int64_t nsamples,
                                 const uint8_t* mask, float* out) {
  for (int64_t s = blockIdx.x; s < nsamples; s += gridDim.x) {
    const float v = vals[s];
    const int64_t b = cu[s], e = cu[s + 1];
    for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x)
      out[t] = (mask == nullptr || mask[t]) ? v : 0.f;
  }
}

// ----------------------------------------------------------------- GAE ----
// State flowing right-to-left: (A_next, V_next).  A valid token maps it to
//   A' = gl*A + g*V + (r - v),  V' = v      ->  M = [[gl, g], [0, 0]], o = (r-v, v)
// a masked token is the identity.  Maps compose by warp scan (fp64).
struct Aff {
  double a, b, k, p, q;  // M = [[a, b], [0, k]], offset (p, q)
};
__device__ __forceinline__ Aff compose(const Aff& F, const Aff& G) {  // F after G
  return Aff{F.a * G.a, F.a * G.b + F.b * G.k, F.k * G.k, F.a * G.p + F.b * G.q + F.p,
             F.k * G.q + F.q};
}
__device__ __forceinline__ Aff shfl_down_aff(const Aff& x, int d) {
  return Aff{__shfl_down_sync(0xffffffffu, x.a, d), __shfl_down_sync(0xffffffffu, x.b, d),
             __shfl_down_sync(0xffffffffu, x.k, d), __shfl_down_sync(0xffffffffu, x.p, d),
             __shfl_down_sync(0xffffffffu, x.q, d)};
}

// One CTA per sequence.  A segment of up to kGaeSeg tokens is staged in
// shared memory with coalesced loads (padded [thread][token] layout, no bank
// conflicts); thread i owns kGaeTpt contiguous tokens: it composes their maps
// right-to-left, a block scan (warp shuffles + smem across warps) gives every
// thread the composite of everything to its right, then it replays its tokens
// with the incoming state, writes A/R back to smem, and the CTA stores them
// coalesced.  Longer sequences loop over segments right-to-left with a carry.
constexpr int kGaeThreads = 256;
constexpr int kGaeTpt = 16;
constexpr int kGaeSeg = kGaeThreads * kGaeTpt;
constexpr int kGaePad = kGaeTpt + 1;

__device__ __forceinline__ int gae_slot(int idx) { return (idx / kGaeTpt) * kGaePad + idx % kGaeTpt; }

__global__ void __launch_bounds__(kGaeThreads) gae_kernel(
    const float* values, const float* rewards, const uint8_t* mask, const int64_t* cu,
    int64_t nseq, double gamma, double lam, float* adv, float* ret) {
  __shared__ float sv[kGaeThreads * kGaePad];
  __shared__ float sr[kGaeThreads * kGaePad];
  __shared__ uint8_t sm[kGaeThreads * kGaePad];
  __shared__ Aff wtot[kGaeThreads / 32];
  __shared__ double carry[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double gl = gamma * lam;
  for (int64_t s = blockIdx.x; s < nseq; s += gridDim.x) {
    const int64_t b = cu[s], e = cu[s + 1];
    double cA = 0.0, cV = 0.0;  // state entering from the right of the segment
    for (int64_t hi = e; hi > b; hi -= kGaeSeg) {
      const int64_t lo = max64(b, hi - kGaeSeg);
      const int n = int(hi - lo);
#pragma unroll 8
      for (int i = tid; i < n; i += kGaeThreads) {  // unrolled: many loads in flight
        const int k = gae_slot(i);
        sv[k] = __ldg(values + lo + i);
        sr[k] = __ldg(rewards + lo + i);
        sm[k] = mask == nullptr ? uint8_t(1) : __ldg(mask + lo + i);
      }
      __syncthreads();
      // this thread's tokens [t0, t1) within the segment
      const int t0 = tid * kGaeTpt, t1 = min(n, t0 + kGaeTpt);
      Aff f{1.0, 0.0, 1.0, 0.0, 0.0};
      for (int t = t1 - 1; t >= t0; --t) {
        const int k = gae_slot(t);
        if (sm[k]) {
          const double v = sv[k];
          f = Aff{gl * f.a, gl * f.b + gamma * f.k, 0.0, gl * f.p + gamma * f.q + (double(sr[k]) - v),
                  v};
        }
      }
      // exclusive composite of the threads to the right: inclusive warp scan
      // from the right, then compose with the totals of later warps
      Aff inc = f;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const Aff o = shfl_down_aff(inc, d);
        if (lane + d < 32) inc = compose(inc, o);
      }
      if (lane == 0) wtot[warp] = inc;
      __syncthreads();
      Aff right{1.0, 0.0, 1.0, 0.0, 0.0};  // composite of later warps
      for (int w = kGaeThreads / 32 - 1; w > warp; --w) right = compose(wtot[w], right);
      Aff ex = shfl_down_aff(inc, 1);      // lanes to my right in this warp
      if (lane == 31) ex = Aff{1.0, 0.0, 1.0, 0.0, 0.0};
      ex = compose(ex, right);
      double A = ex.a * cA + ex.b * cV + ex.p;
      double Vn = ex.k * cV + ex.q;
      for (int t = t1 - 1; t >= t0; --t) {
        const int k = gae_slot(t);
        const double v = sv[k];
        if (sm[k]) {
          A = (double(sr[k]) - v) + gamma * Vn + gl * A;
          Vn = v;
        }
        sv[k] = float(A);      // advantage
        sr[k] = float(A + v);  // return
      }
      if (tid == 0) {
        carry[0] = A;
        carry[1] = Vn;
      }
      __syncthreads();
      for (int i = tid; i < n; i += kGaeThreads) {
        const int k = gae_slot(i);
        adv[lo + i] = sv[k];
        ret[lo + i] = sr[k];
      }
      cA = carry[0];
      cV = carry[1];
      __syncthreads();
    }
  }
}

// ------------------------------------------------------- masked moments ----
__global__ void moments_partial_kernel(const float* x, const uint8_t* mask, int64_t n,
                                       double* part) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(n, lo + per);
  double c = 0, s = 0, q = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (mask == nullptr || mask[i]) {
      const double v = x[i];
      c += 1.0;
      s += v;
      q += v * v;
    }
  }
  __shared__ double red[3][32];
  c = warp_sum(c);
  s = warp_sum(s);
  q = warp_sum(q);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][w] = c;
    red[1][w] = s;
    red[2][w] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, bsum = 0, cc = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) {
      a += red[0][i];
      bsum += red[1][i];
      cc += red[2][i];
    }
    part[3 * blockIdx.x + 0] = a;
    part[3 * blockIdx.x + 1] = bsum;
    part[3 * blockIdx.x + 2] = cc;
  }
}

__global__ void moments_final_kernel(const double* part, int nparts, double* out) {
  if (threadIdx.x != 0) return;
  double a = 0, b = 0, c = 0;
  for (int i = 0; i < nparts; ++i) {
    a += part[3 * i];
    b += part[3 * i + 1];
    c += part[3 * i + 2];
  }
  out[0] = a;
  out[1] = b;
  out[2] = c;
}

__global__ void whiten_kernel(float* x, const uint8_t* mask, int64_t n, const double* mom,
                              int32_t shift_mean) {
  const double cnt = mom[0];
  const double mean = cnt > 0 ? mom[1] / cnt : 0.0;
  const double var = cnt > 1 ? (mom[2] - mom[1] * mean) / (cnt - 1.0) : 0.0;
  const double inv = 1.0 / sqrt(var + 1e-8);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (mask == nullptr || mask[i]) {
      double v = (double(x[i]) - mean) * inv;
      if (!shift_mean) v += mean;
      x[i] = float(v);
    }
  }
}

}  // namespace

int64_t grpo_num_local_groups(int64_t n, uint64_t first_id, int32_t G) {
  if (n <= 0 || G <= 0) return 0;
  return int64_t((first_id + uint64_t(n) - 1) / uint64_t(G) - first_id / uint64_t(G) + 1);
}

int grpo_moments_launch(const float* r, int64_t n, uint64_t first_id, int32_t G, double* out,
                        cudaStream_t st) {
  YATT_REQUIRE(G > 0, YATT_ERR_CONFIG, "grpo: group_size must be positive");
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "grpo: n_samples must be >= 0");
  const int64_t ng = grpo_num_local_groups(n, first_id, G);
  if (ng == 0) return YATT_OK;
  grpo_moments_kernel<<<unsigned(ceil_div(ng, 128)), 128, 0, st>>>(r, n, first_id, G, ng, out);
  return check_launch("grpo_moments_kernel");
}

int grpo_adv_launch(const float* r, int64_t n, uint64_t first_id, int32_t G, float eps,
                    int32_t norm_by_std, const double* moments, float* adv, cudaStream_t st) {
  YATT_REQUIRE(G > 0, YATT_ERR_CONFIG, "grpo: group_size must be positive");
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "grpo: n_samples must be >= 0");
  YATT_REQUIRE(eps >= 0.f, YATT_ERR_CONFIG, "grpo: eps must be >= 0");
  if (n == 0) return YATT_OK;
  grpo_adv_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(r, n, first_id, G, eps,
                                                              norm_by_std, moments, adv);
  return check_launch("grpo_adv_kernel");
}

int broadcast_launch(const float* vals, const int64_t* cu, int64_t nsamples, const uint8_t* mask,
                     float* out, cudaStream_t st) {
  YATT_REQUIRE(nsamples >= 0, YATT_ERR_CONFIG, "broadcast: n_samples must be >= 0");
  if (nsamples == 0) return YATT_OK;
  const int grid = int(min64(nsamples, int64_t(num_sms()) * 8));
  broadcast_kernel<<<grid, 256, 0, st>>>(vals, cu, nsamples, mask, out);
  return check_launch("broadcast_kernel");
}

int gae_launch(const float* values, const float* rewards, const uint8_t* mask, const int64_t* cu,
               int64_t nseq, float gamma, float lam, float* adv, float* ret, cudaStream_t st) {
  YATT_REQUIRE(nseq >= 0, YATT_ERR_CONFIG, "gae: n_seqs must be >= 0");
  YATT_REQUIRE(gamma >= 0.f && lam >= 0.f, YATT_ERR_CONFIG, "gae: gamma/lam must be >= 0");
  if (nseq == 0) return YATT_OK;
  const int grid = int(min64(nseq, int64_t(num_sms()) * 8));
  gae_kernel<<<grid, kGaeThreads, 0, st>>>(values, rewards, mask, cu, nseq, double(gamma),
                                           double(lam), adv, ret);
  return check_launch("gae_kernel");
}

size_t moments_workspace_bytes() { return size_t(3) * 2 * 160 * sizeof(double); }

int masked_moments_launch(const float* x, const uint8_t* mask, int64_t n, double* out,
                          double* ws, cudaStream_t st) {
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "moments: n must be >= 0");
  const int parts = min(2 * num_sms(), 320);
  moments_partial_kernel<<<parts, 256, 0, st>>>(x, mask, n, ws);
  int rc = check_launch("moments_partial_kernel");
  if (rc) return rc;
  moments_final_kernel<<<1, 32, 0, st>>>(ws, parts, out);
  return check_launch("moments_final_kernel");
}

int whiten_launch(float* x, const uint8_t* mask, int64_t n, const double* mom, int32_t shift,
                  cudaStream_t st) {
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "whiten: n must be >= 0");
  if (n == 0) return YATT_OK;
  const int grid = int(min64(ceil_div(n, 256), int64_t(num_sms()) * 8));
  whiten_kernel<<<grid, 256, 0, st>>>(x, mask, n, mom, shift);
  return check_launch("whiten_kernel");
}

}  // namespace yattb
