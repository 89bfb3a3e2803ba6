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

__device__ __forceinline__ float bcast_val(float v, const uint8_t* mask, int64_t t) {
  return (mask == nullptr || mask[t]) ? v : 0.f;
}

// One CTA per sample: scalar head to the first 4-aligned token, 16-byte
// streaming stores over the body (out 16-B aligned, mask read as u32), tail.
template <bool kVec>
__global__ void broadcast_kernel(const float* vals, const int64_t* cu, int64_t nsamples,
                                 const uint8_t* mask, float* out) {
  for (int64_t s = blockIdx.x; s < nsamples; s += gridDim.x) {
    const float v = vals[s];
    const int64_t b = cu[s], e = cu[s + 1];
    if (!kVec) {
      for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) out[t] = bcast_val(v, mask, t);
      continue;
    }
    const int64_t hb = min64(e, (b + 3) & ~int64_t(3));
    const int64_t jb = hb >> 2, je = max64(jb, e >> 2);
    if (b + int64_t(threadIdx.x) < hb) out[b + threadIdx.x] = bcast_val(v, mask, b + threadIdx.x);
    for (int64_t j = jb + threadIdx.x; j < je; j += blockDim.x) {
      float4 o = make_float4(v, v, v, v);
      if (mask != nullptr) {
        const uint32_t m = __ldg(reinterpret_cast<const uint32_t*>(mask + 4 * j));
        o.x = (m & 0xffu) ? v : 0.f;
        o.y = (m & 0xff00u) ? v : 0.f;
        o.z = (m & 0xff0000u) ? v : 0.f;
        o.w = (m & 0xff000000u) ? v : 0.f;
      }
      __stcs(reinterpret_cast<float4*>(out + 4 * j), o);
    }
    const int64_t tb = max64(hb, 4 * je);
    if (tb + int64_t(threadIdx.x) < e) out[tb + threadIdx.x] = bcast_val(v, mask, tb + threadIdx.x);
  }
}

// ----------------------------------------------------------------- GAE ----
// State flowing right-to-left: (A_next, V_next).  A valid token maps it to
//   A' = gl*A + g*V + (r - v),  V' = v      ->  M = [[gl, g], [0, 0]], o = (r-v, v)
// a masked token is the identity; the last token of a sequence first resets
// the state to (0, 0) (the zero map).  Maps compose associatively (fp64).
struct Aff {
  double a, b, k, p, q;  // M = [[a, b], [0, k]], offset (p, q)
};
__device__ __forceinline__ Aff aff_id() { return Aff{1.0, 0.0, 1.0, 0.0, 0.0}; }
__device__ __forceinline__ Aff compose(const Aff& F, const Aff& G) {  // F after G
  return Aff{F.a * G.a, F.a * G.b + F.b * G.k, F.k * G.k, F.a * G.p + F.b * G.q + F.p,
             F.k * G.q + F.q};
}
__device__ __forceinline__ Aff shfl_down_aff(const Aff& x, int d) {
  return Aff{__shfl_down_sync(0xffffffffu, x.a, d), __shfl_down_sync(0xffffffffu, x.b, d),
             __shfl_down_sync(0xffffffffu, x.k, d), __shfl_down_sync(0xffffffffu, x.p, d),
             __shfl_down_sync(0xffffffffu, x.q, d)};
}

// Single-pass scan over the packed token array with decoupled look-back,
// one 512-token tile per warp (lane l owns 16 contiguous tokens).  Warps
// claim tiles right to left by an atomic ticket: a tile only waits on tiles
// with earlier tickets, whose warps are running, so the smallest unfinished
// ticket always progresses and the scan cannot deadlock.  Bytes: 9 read + 8
// written per token, once (+1 bit per token for the sequence-end mask).
constexpr int kGaeTpt = 16;
constexpr int kGaeWTile = 32 * kGaeTpt;

// Device workspace (yatt_gae_workspace_bytes), zeroed per call:
//   ticket | rec[ntiles] (16 B each) | ends[ntiles * 16] (bit i: token i is
//   the last token of a sequence).
struct GaeWs {
  uint32_t* ticket;
  uint4* rec;
  uint32_t* ends;
  double* mom;  // [ntiles][3] masked (count, sum, sum^2) of the stored advantages
};
__host__ __device__ inline size_t gae_align(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline GaeWs gae_ws(void* base, int64_t ntiles) {
  uint8_t* b = static_cast<uint8_t*>(base);
  const size_t mom_off = gae_align(16 + 16 * size_t(ntiles) + 64 * size_t(ntiles));
  return GaeWs{reinterpret_cast<uint32_t*>(b), reinterpret_cast<uint4*>(b + 16),
               reinterpret_cast<uint32_t*>(b + 16 + 16 * size_t(ntiles)),
               reinterpret_cast<double*>(b + mom_off)};
}
size_t gae_ws_bytes(int64_t ntiles) {
  return gae_align(16 + 16 * size_t(ntiles) + 64 * size_t(ntiles)) + 24 * size_t(ntiles);
}

struct GaeArgs {
  const float* values;
  const float* rewards;
  const uint8_t* mask;
  const int64_t* cu;
  int64_t nseq, n_tokens, ntiles;
  double gamma, lam;
  float* adv;
  float* ret;
};

__device__ __forceinline__ uint4 ld_incl(const uint4* p) {
  uint4 w;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "l"(p)
               : "memory");
  return w;
}

// Tile record (one 16-byte word per tile, written once with a single store,
// so data and flag arrive together and no fence is needed; both kinds depend
// only on the tile's own tokens, so every look-back composes the same maps in
// the same order: the scan is run-to-run bit-deterministic):
//   flag 2: {double A, float V}     tile holding a sequence end: the state it
//                                   passes to the left (constant composite)
//   flag 1: {double p, float q, m}  tile without one: its composite, m valid
//           tokens -> a = gl^m, b = g gl^(m-1), k = 0 (m = 0: identity)
__device__ __forceinline__ void st_rec(uint4* p, double x, double y, uint32_t tag) {
  const uint4 w = make_uint4(uint32_t(__double2loint(x)), uint32_t(__double2hiint(x)),
                             __float_as_uint(float(y)), tag);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w.x), "r"(w.y),
               "r"(w.z), "r"(w.w)
               : "memory");
}
__device__ __forceinline__ double ipow(double x, uint32_t m) {
  double r = 1.0;
  while (m) {
    if (m & 1u) r *= x;
    x *= x;
    m >>= 1;
  }
  return r;
}
__device__ __forceinline__ Aff rec_map(const uint4& w, double gamma, double gl) {
  const double x = __hiloint2double(int(w.y), int(w.x)), y = double(__uint_as_float(w.z));
  if ((w.w & 3u) == 2u) return Aff{0.0, 0.0, 0.0, x, y};
  const uint32_t m = w.w >> 2;
  if (m == 0u) return aff_id();
  return Aff{ipow(gl, m), gamma * ipow(gl, m - 1u), 0.0, x, y};
}

// ---- the scan kernel: one 512-token tile per warp, no CTA barriers ----
// Lane l owns tokens [lo + 16l, lo + 16l + 16) in registers (float4 loads)
// and their 16 sequence-end bits; lanes whose 16 tokens are all inside, valid
// and not sequence ends take a straight-line fp64 path.  Compose, shuffle
// scan, publish the tile record, then the look-back reads 32 predecessor
// records at once (lane i -> tile t+1+i) and composes them up to the first
// tile holding a sequence end with one shuffle tree: one L2 round trip per 32
// tiles, and no tile waits on another tile's look-back.
__device__ __forceinline__ Aff shfl_aff(const Aff& x, int src) {
  return Aff{__shfl_sync(0xffffffffu, x.a, src), __shfl_sync(0xffffffffu, x.b, src),
             __shfl_sync(0xffffffffu, x.k, src), __shfl_sync(0xffffffffu, x.p, src),
             __shfl_sync(0xffffffffu, x.q, src)};
}

#ifdef YATT_GAE_PROFILE
// Phase timestamps per tile (variant builds only; tools/gae_phases.py):
// start, ticket, ends/data, scan done, carry known, tile done.
__device__ long long g_gae_prof[16384][6];
#define GAE_WSTAMP(k) \
  if (lane == 0 && t >= 0 && t < 16384) g_gae_prof[t][k] = clock64()
#else
#define GAE_WSTAMP(k)
#endif

// Marks the last token of every non-empty sequence in the ends bitmask.
__global__ void gae_mark_ends_kernel(const int64_t* cu, int64_t nseq, int64_t n_tokens,
                                     uint32_t* ends) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nseq) return;
  const int64_t b = __ldg(cu + k), e = min64(__ldg(cu + k + 1), n_tokens);
  if (e > b && e >= 1) atomicOr(ends + ((e - 1) >> 5), 1u << ((e - 1) & 31));
}

#ifndef YATT_GAE_MINB  // 6 CTAs/SM (80 regs, no spills): 59 us vs 64 us at 5 (96 regs); 7 / 8 (spilling) no faster
#define YATT_GAE_MINB 6
#endif
// kMom: also the masked moments (count, sum, sum^2) of the advantages it
// stores, one fp64 partial per tile (whitening without a second pass).
// (The scalar-load form for unaligned views keeps 4 CTAs/SM: at 6 its extra
// address registers spilled.)
template <bool kVec, bool kMom>
__global__ void __launch_bounds__(128, kVec ? YATT_GAE_MINB : 4) gae_warp_kernel(const GaeArgs g,
                                                                                 GaeWs ws) {
  const int lane = threadIdx.x & 31;
  const double gamma = g.gamma, gl = g.gamma * g.lam;
  int64_t t = 0;
#ifdef YATT_GAE_PROFILE
  const long long t_start = clock64();
#endif
  if (lane == 0) t = g.ntiles - 1 - int64_t(atomicAdd(ws.ticket, 1u));
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t < 0) return;
#ifdef YATT_GAE_PROFILE
  if (lane == 0 && t < 16384) g_gae_prof[t][0] = t_start;
#endif
  GAE_WSTAMP(1);
  const int64_t lo = t * kGaeWTile, hi = min64(g.n_tokens, lo + kGaeWTile);
  const int64_t x0 = lo + int64_t(lane) * kGaeTpt;
  const int nmine = int(max64(0, min64(kGaeTpt, hi - x0)));
  // loads first: they fly while the sequence ends are found
  float v[kGaeTpt], r[kGaeTpt];
  uint32_t validm = 0xffffu;
  if (kVec && nmine == kGaeTpt) {
#pragma unroll
    for (int q = 0; q < kGaeTpt / 4; ++q) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(g.values + x0) + q);
      const float4 b = __ldcs(reinterpret_cast<const float4*>(g.rewards + x0) + q);
      v[4 * q] = a.x, v[4 * q + 1] = a.y, v[4 * q + 2] = a.z, v[4 * q + 3] = a.w;
      r[4 * q] = b.x, r[4 * q + 1] = b.y, r[4 * q + 2] = b.z, r[4 * q + 3] = b.w;
    }
    if (g.mask) {
      const uint4 m4 = __ldcs(reinterpret_cast<const uint4*>(g.mask + x0));
      const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
      validm = 0u;
#pragma unroll
      for (int j = 0; j < kGaeTpt; ++j)
        validm |= ((mw[j >> 2] >> (8 * (j & 3))) & 0xffu) ? (1u << j) : 0u;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kGaeTpt; ++j) {
      v[j] = j < nmine ? g.values[x0 + j] : 0.f;
      r[j] = j < nmine ? g.rewards[x0 + j] : 0.f;
    }
    if (g.mask) {
      validm = 0u;
#pragma unroll
      for (int j = 0; j < kGaeTpt; ++j) validm |= (j < nmine && g.mask[x0 + j]) ? (1u << j) : 0u;
    }
  }
  // this lane's 16 sequence-end bits (marked by gae_mark_ends_kernel)
  const uint32_t lb = (__ldcg(ws.ends + (x0 >> 5)) >> (x0 & 31)) & 0xffffu;
  const int64_t in_lo = __ldg(g.cu), in_hi = min64(g.n_tokens, __ldg(g.cu + g.nseq));
  GAE_WSTAMP(2);
  uint32_t insm = 0u;
  {
    const int64_t a = max64(0, in_lo - x0), b = min64(nmine, in_hi - x0);
    if (b > a) insm = ((1u << b) - 1u) & ~((1u << a) - 1u);
  }
  // compose this lane's tokens right to left.  Fast path (most lanes): all 16
  // tokens inside, valid and not sequence ends -> a = gl^16, b = g gl^15,
  // k = 0 and only the offset chain is computed.
  const bool plain = insm == 0xffffu && validm == 0xffffu && lb == 0u;
  Aff f = aff_id();
  if (plain) {
    double p = 0.0, q = 0.0;
#pragma unroll
    for (int j = kGaeTpt - 1; j >= 0; --j) {
      const double vv = double(v[j]);
      p = fma(gl, p, fma(gamma, q, double(r[j]) - vv));
      q = vv;
    }
    double a = gl, b = gamma;
#pragma unroll
    for (int j = 1; j < kGaeTpt; ++j) a *= gl, b *= gl;
    f = Aff{a, b, 0.0, p, q};
  } else {
#pragma unroll
    for (int j = kGaeTpt - 1; j >= 0; --j) {
      const uint32_t bit = 1u << j;
      if (!(insm & bit)) continue;
      if (lb & bit) f = Aff{0.0, 0.0, 0.0, 0.0, 0.0};
      if (validm & bit) {
        const double vv = double(v[j]);
        f = Aff{gl * f.a, gl * f.b + gamma * f.k, 0.0, gl * f.p + gamma * f.q + (double(r[j]) - vv),
                vv};
      }
    }
  }
  // inclusive scan from the right: lane 0 ends with the tile's composite
  Aff inc = f;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Aff o = shfl_down_aff(inc, d);
    if (lane + d < 32) inc = compose(inc, o);
  }
  Aff ex = shfl_down_aff(inc, 1);  // lanes to my right
  if (lane == 31) ex = aff_id();
  const Aff tot = shfl_aff(inc, 0);
  const bool constant = tot.a == 0.0 && tot.b == 0.0 && tot.k == 0.0;
  GAE_WSTAMP(3);
  if (!constant) {  // valid tokens of a tile without sequence ends
    const uint32_t m = __reduce_add_sync(0xffffffffu, uint32_t(__popc(validm & insm)));
    if (lane == 0) st_rec(ws.rec + t, tot.p, tot.q, (m << 2) | 1u);
  } else if (lane == 0) {
    st_rec(ws.rec + t, tot.p, tot.q, 2u);
  }
  // the carry: composite of the tiles to the right up to the first one holding
  // a sequence end (the array end counts as state (0, 0)); one 16-byte record
  // per tile, 32 tiles per round trip
  Aff c = aff_id();
  for (int64_t base = t + 1;; base += 32) {
    const int64_t j = base + lane;
    Aff m = aff_id();
    int first;
    for (int spins = 0;; ++spins) {
      const uint4 w = j < g.ntiles ? ld_incl(ws.rec + j) : make_uint4(0u, 0u, 0u, 2u);
      const uint32_t bi = __ballot_sync(0xffffffffu, (w.w & 3u) == 2u);
      const uint32_t ba = __ballot_sync(0xffffffffu, (w.w & 3u) != 0u);
      first = bi ? __ffs(bi) - 1 : 32;
      const uint32_t need = first == 32 ? 0xffffffffu : ((2u << first) - 1u);
      if ((ba & need) == need) {
        if (lane <= first) m = rec_map(w, gamma, gl);
        break;
      }
      if (spins > 4) __nanosleep(32);
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {  // lane 0: m_0 o m_1 o ... o m_31
      const Aff o = shfl_down_aff(m, d);
      if (lane + d < 32) m = compose(m, o);
    }
    c = compose(c, shfl_aff(m, 0));
    if (first < 32) break;
  }
  const double cA = c.p, cV = c.q;  // c ends in a constant map
  GAE_WSTAMP(4);
  double A = ex.a * cA + ex.b * cV + ex.p;
  double Vn = ex.k * cV + ex.q;
  float ao[kGaeTpt], ro[kGaeTpt];
  double mc = 0.0, ms = 0.0, mq = 0.0;
  if (plain) {
#pragma unroll
    for (int j = kGaeTpt - 1; j >= 0; --j) {
      const double vv = double(v[j]);
      A = (double(r[j]) - vv) + gamma * Vn + gl * A;
      Vn = vv;
      ao[j] = float(A);
      ro[j] = float(A + vv);
      if (kMom) {
        const double af = double(ao[j]);
        ms += af;
        mq += af * af;
      }
    }
    if (kMom) mc = double(kGaeTpt);
  } else {
#pragma unroll
    for (int j = kGaeTpt - 1; j >= 0; --j) {
      const uint32_t bit = 1u << j;
      ao[j] = 0.f, ro[j] = 0.f;
      if (!(insm & bit)) continue;
      if (lb & bit) A = 0.0, Vn = 0.0;
      const double vv = double(v[j]);
      if (validm & bit) {
        A = (double(r[j]) - vv) + gamma * Vn + gl * A;
        Vn = vv;
      }
      ao[j] = float(A);
      ro[j] = float(A + vv);
      if (kMom && (validm & bit)) {
        const double af = double(ao[j]);
        mc += 1.0;
        ms += af;
        mq += af * af;
      }
    }
  }
  if (kMom) {  // fixed-order warp reduction -> this tile's partial
    mc = warp_sum(mc);
    ms = warp_sum(ms);
    mq = warp_sum(mq);
    if (lane == 0) {
      ws.mom[3 * t] = mc;
      ws.mom[3 * t + 1] = ms;
      ws.mom[3 * t + 2] = mq;
    }
  }
  if (kVec && insm == 0xffffu) {
#pragma unroll
    for (int q = 0; q < kGaeTpt / 4; ++q) {
      __stcs(reinterpret_cast<float4*>(g.adv + x0) + q,
             make_float4(ao[4 * q], ao[4 * q + 1], ao[4 * q + 2], ao[4 * q + 3]));
      __stcs(reinterpret_cast<float4*>(g.ret + x0) + q,
             make_float4(ro[4 * q], ro[4 * q + 1], ro[4 * q + 2], ro[4 * q + 3]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < kGaeTpt; ++j)
      if (insm & (1u << j)) {
        g.adv[x0 + j] = ao[j];
        g.ret[x0 + j] = ro[j];
      }
  }
  GAE_WSTAMP(5);
}


// ------------------------------------------------------- masked moments ----
constexpr int kMomThreads = 256;
constexpr int kMomMaxParts = 640;

__device__ __forceinline__ void mom_add(float x, bool valid, double& c, double& s, double& q) {
  if (valid) {
    const double v = double(x);
    c += 1.0;
    s += v;
    q += v * v;
  }
}
__device__ __forceinline__ void mom_add4(const float4& x, uint32_t m, double& c, double& s,
                                         double& q) {
  mom_add(x.x, m & 0xffu, c, s, q);
  mom_add(x.y, m & 0xff00u, c, s, q);
  mom_add(x.z, m & 0xff0000u, c, s, q);
  mom_add(x.w, m & 0xff000000u, c, s, q);
}
__device__ __forceinline__ uint32_t mask4(const uint8_t* mask, int64_t j) {
  return mask == nullptr ? 0x01010101u : __ldg(reinterpret_cast<const uint32_t*>(mask + 4 * j));
}

// Contiguous ranges of 4-element vectors per block, two in flight per thread;
// the n % 4 tail goes to the last block.  fp64 (count, sum, sum of squares).
template <bool kVec>
__global__ void __launch_bounds__(kMomThreads) moments_partial_kernel(const float* x,
                                                                      const uint8_t* mask,
                                                                      int64_t n, double* part) {
  double c = 0, s = 0, q = 0;
  if (kVec) {
    const int64_t nv = n >> 2;
    const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
    const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(nv, lo + per);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    int64_t j = lo + threadIdx.x;
    for (; j + kMomThreads < hi; j += 2 * kMomThreads) {
      const float4 a = __ldg(x4 + j), b = __ldg(x4 + j + kMomThreads);
      const uint32_t ma = mask4(mask, j), mb = mask4(mask, j + kMomThreads);
      mom_add4(a, ma, c, s, q);
      mom_add4(b, mb, c, s, q);
    }
    if (j < hi) mom_add4(__ldg(x4 + j), mask4(mask, j), c, s, q);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < (n & 3)) {
      const int64_t i = 4 * nv + threadIdx.x;
      mom_add(x[i], mask == nullptr || mask[i], c, s, q);
    }
  } else {
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = int64_t(blockIdx.x) * per, hi = min64(n, lo + per);
    for (int64_t i = lo + threadIdx.x; i < hi; i += kMomThreads)
      mom_add(x[i], mask == nullptr || mask[i], c, s, q);
  }
  __shared__ double red[3][kMomThreads / 32];
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
    for (int i = 0; i < kMomThreads / 32; ++i) {
      a += red[0][i];
      bsum += red[1][i];
      cc += red[2][i];
    }
    part[3 * blockIdx.x + 0] = a;
    part[3 * blockIdx.x + 1] = bsum;
    part[3 * blockIdx.x + 2] = cc;
  }
}

struct WhitenCoef {
  double mean, inv;
};
__device__ __forceinline__ WhitenCoef whiten_coef(const double* mom) {
  const double cnt = mom[0];
  const double mean = cnt > 0 ? mom[1] / cnt : 0.0;
  const double var = cnt > 1 ? (mom[2] - mom[1] * mean) / (cnt - 1.0) : 0.0;
  return WhitenCoef{mean, 1.0 / sqrt(var + 1e-8)};
}
__device__ __forceinline__ float whiten1(float x, const WhitenCoef& w, int32_t shift_mean) {
  double v = (f2d_int(x) - w.mean) * w.inv;
  if (!shift_mean) v += w.mean;
  return float(v);
}

template <bool kVec>
__global__ void whiten_kernel(float* x, const uint8_t* mask, int64_t n, const double* mom,
                              int32_t shift_mean) {
  const WhitenCoef w = whiten_coef(mom);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kVec) {
    const int64_t nv = n >> 2;
    float4* x4 = reinterpret_cast<float4*>(x);
    for (int64_t j = t0; j < nv; j += stride) {
      float4 a = x4[j];
      const uint32_t m = mask4(mask, j);
      if (m & 0xffu) a.x = whiten1(a.x, w, shift_mean);
      if (m & 0xff00u) a.y = whiten1(a.y, w, shift_mean);
      if (m & 0xff0000u) a.z = whiten1(a.z, w, shift_mean);
      if (m & 0xff000000u) a.w = whiten1(a.w, w, shift_mean);
      x4[j] = a;
    }
    if (t0 < (n & 3)) {
      const int64_t i = 4 * nv + t0;
      if (mask == nullptr || mask[i]) x[i] = whiten1(x[i], w, shift_mean);
    }
  } else {
    for (int64_t i = t0; i < n; i += stride)
      if (mask == nullptr || mask[i]) x[i] = whiten1(x[i], w, shift_mean);
  }
}

bool vec_ok(const void* f32, const uint8_t* mask) {
  return (reinterpret_cast<uintptr_t>(f32) & 15) == 0 && (reinterpret_cast<uintptr_t>(mask) & 3) == 0;
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
  if (vec_ok(out, mask))
    broadcast_kernel<true><<<grid, 256, 0, st>>>(vals, cu, nsamples, mask, out);
  else
    broadcast_kernel<false><<<grid, 256, 0, st>>>(vals, cu, nsamples, mask, out);
  return check_launch("broadcast_kernel");
}

size_t gae_workspace_bytes(int64_t n_tokens) {
  return gae_ws_bytes(ceil_div(max64(n_tokens, 0), kGaeWTile));
}

int gae_launch(const float* values, const float* rewards, const uint8_t* mask, const int64_t* cu,
               int64_t nseq, int64_t n_tokens, float gamma, float lam, float* adv, float* ret,
               void* ws, size_t ws_bytes, cudaStream_t st, double* moments) {
  YATT_REQUIRE(nseq >= 0 && n_tokens >= 0, YATT_ERR_CONFIG, "gae: n_seqs and n_tokens must be >= 0");
  YATT_REQUIRE(gamma >= 0.f && lam >= 0.f, YATT_ERR_CONFIG, "gae: gamma/lam must be >= 0");
  if (nseq == 0 || n_tokens == 0) {
    if (moments) YATT_TRY_CUDA(cudaMemsetAsync(moments, 0, 3 * sizeof(double), st));
    return YATT_OK;
  }
  YATT_REQUIRE(values && rewards && cu && adv && ret, YATT_ERR_CONFIG, "gae: null pointer");
  const int64_t ntiles = ceil_div(n_tokens, kGaeWTile);
  YATT_REQUIRE(ws != nullptr && ws_bytes >= gae_ws_bytes(ntiles), YATT_ERR_WORKSPACE,
               "gae: workspace too small (%zu < %zu)", ws_bytes, gae_ws_bytes(ntiles));
  YATT_REQUIRE(ntiles < (int64_t(1) << 31), YATT_ERR_CONFIG, "gae: too many tokens");
  YATT_TRY_CUDA(cudaMemsetAsync(ws, 0, gae_ws_bytes(ntiles), st));
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool vec = a16(values) && a16(rewards) && a16(mask) && a16(adv) && a16(ret);
  const GaeArgs args{values, rewards, mask, cu, nseq, n_tokens, ntiles, double(gamma), double(lam),
                     adv, ret};
  const GaeWs w = gae_ws(ws, ntiles);
  gae_mark_ends_kernel<<<unsigned(ceil_div(nseq, 256)), 256, 0, st>>>(cu, nseq, n_tokens, w.ends);
  const unsigned grid = unsigned(ceil_div(ntiles, 4));  // 4 warps = 4 tiles per CTA
  if (moments) {
    if (vec)
      gae_warp_kernel<true, true><<<grid, 128, 0, st>>>(args, w);
    else
      gae_warp_kernel<false, true><<<grid, 128, 0, st>>>(args, w);
    const int rc = check_launch("gae_kernel");
    if (rc) return rc;
    reduce_parts_kernel<3><<<1, 256, 0, st>>>(w.mom, int(ntiles), moments);
    return check_launch("reduce_parts_kernel<3>");
  }
  if (vec)
    gae_warp_kernel<true, false><<<grid, 128, 0, st>>>(args, w);
  else
    gae_warp_kernel<false, false><<<grid, 128, 0, st>>>(args, w);
  return check_launch("gae_kernel");
}

size_t moments_workspace_bytes() { return size_t(3) * kMomMaxParts * sizeof(double); }

int masked_moments_launch(const float* x, const uint8_t* mask, int64_t n, double* out,
                          double* ws, cudaStream_t st) {
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "moments: n must be >= 0");
  const int parts = min(4 * num_sms(), kMomMaxParts);
  if (vec_ok(x, mask))
    moments_partial_kernel<true><<<parts, kMomThreads, 0, st>>>(x, mask, n, ws);
  else
    moments_partial_kernel<false><<<parts, kMomThreads, 0, st>>>(x, mask, n, ws);
  int rc = check_launch("moments_partial_kernel");
  if (rc) return rc;
  reduce_parts_kernel<3><<<1, 256, 0, st>>>(ws, parts, out);
  return check_launch("reduce_parts_kernel<3>");
}

int whiten_launch(float* x, const uint8_t* mask, int64_t n, const double* mom, int32_t shift,
                  cudaStream_t st) {
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "whiten: n must be >= 0");
  if (n == 0) return YATT_OK;
  const int grid = int(min64(ceil_div(ceil_div(n, 4), 256), int64_t(num_sms()) * 8));
  if (vec_ok(x, mask))
    whiten_kernel<true><<<grid, 256, 0, st>>>(x, mask, n, mom, shift);
  else
    whiten_kernel<false><<<grid, 256, 0, st>>>(x, mask, n, mom, shift);
  return check_launch("whiten_kernel");
}

}  // namespace yattb

#ifdef YATT_GAE_PROFILE
extern "C" int yatt_debug_gae_profile(long long* out, int ntiles) {
  return int(cudaMemcpyFromSymbol(out, yattb::g_gae_prof, sizeof(long long) * 6 *
                                                            size_t(ntiles < 16384 ? ntiles : 16384)));
}
#endif
