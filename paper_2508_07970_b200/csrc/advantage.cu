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

// Single-pass scan over the packed token array with decoupled look-back.
// The array is cut into 2,048-token tiles; thread i of a 128-thread CTA owns
// 16 contiguous tokens.  Persistent CTAs claim tiles right to left by an
// atomic ticket (a tile only waits on tiles with earlier tickets, whose
// holders are running: the smallest unfinished ticket is always being
// processed, so the scan cannot deadlock) and keep the NEXT tile's values,
// rewards and mask in flight (cp.async.bulk into the other shared-memory
// stage) while the current tile is scanned.  Each tile publishes its
// composite map (flag 1) and, once its incoming state is known, its outgoing
// state (flag 2); a tile holding a sequence end has a constant composite and
// publishes flag 2 at once, so look-back chains stop at the first sequence
// boundary.  Bytes: 9 read + 8 written per token, once.
constexpr int kGaeThreads = 128;
constexpr int kGaeTpt = 16;
constexpr int kGaeTile = kGaeThreads * kGaeTpt;

// Device workspace (yatt_gae_workspace_bytes): ticket | incl[ntiles] |
// aflag[ntiles] (zeroed per call) | agg[ntiles].  incl[t] is one 16-byte
// record {double A; float V; u32 flag}: the state leaving tile t to the left
// (V is an input value or 0, so fp32 holds it exactly) and its ready flag in
// the same single 16-byte store, so a look-back step is one L2 round trip.
struct GaeWs {
  uint32_t* ticket;
  uint4* incl;      // [ntiles]
  uint32_t* aflag;  // [ntiles] agg[t] published
  Aff* agg;         // [ntiles] composite map of tile t
};
__host__ __device__ inline size_t gae_align(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline GaeWs gae_ws(void* base, int64_t ntiles) {
  uint8_t* b = static_cast<uint8_t*>(base);
  GaeWs w;
  w.ticket = reinterpret_cast<uint32_t*>(b);
  w.incl = reinterpret_cast<uint4*>(b + 16);
  w.aflag = reinterpret_cast<uint32_t*>(b + 16 + 16 * size_t(ntiles));
  w.agg = reinterpret_cast<Aff*>(b + gae_align(16 + 20 * size_t(ntiles)));
  return w;
}
size_t gae_ws_bytes(int64_t ntiles) {
  return gae_align(16 + 20 * size_t(ntiles)) + sizeof(Aff) * size_t(ntiles);
}
size_t gae_zero_bytes(int64_t ntiles) { return 16 + 20 * size_t(ntiles); }

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_incl(uint4* p, double A, double V) {
  const uint4 w = make_uint4(uint32_t(__double2loint(A)), uint32_t(__double2hiint(A)),
                             __float_as_uint(float(V)), 2u);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w.x), "r"(w.y),
               "r"(w.z), "r"(w.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_incl(const uint4* p) {
  uint4 w;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "l"(p)
               : "memory");
  return w;
}

// First index k in [k0, k1) with a[k] >= key (k1 if none), a non-decreasing;
// one warp, 32-ary: positions >= k1 count as +inf, so the predicate is
// monotone in the lane and the answer stays inside [k0, k1].
__device__ int64_t warp_lower_bound(const int64_t* a, int64_t k0, int64_t k1, int64_t key,
                                    int lane) {
  while (k1 - k0 > 32) {
    const int64_t step = (k1 - k0 + 31) / 32;
    const int64_t idx = k0 + lane * step;
    const bool ge = idx >= k1 || __ldg(a + idx) >= key;
    const uint32_t bal = __ballot_sync(0xffffffffu, ge);
    if (bal & 1u) return k0;
    const int f = bal ? __ffs(bal) - 1 : 32;
    const int64_t nk0 = k0 + int64_t(f - 1) * step + 1;
    if (f < 32) k1 = min64(k1, k0 + int64_t(f) * step);
    k0 = nk0;
  }
  const bool ge = k0 + lane < k1 && __ldg(a + k0 + lane) >= key;
  const uint32_t bal = __ballot_sync(0xffffffffu, ge);
  return bal ? k0 + __ffs(bal) - 1 : k1;
}

struct __align__(128) GaeStage {
  float v[kGaeTile];
  float r[kGaeTile];
  uint8_t m[kGaeTile];
};

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

#ifdef YATT_GAE_PROFILE
// Phase timestamps per tile (variant builds only): start, data ready, ends
// marked, scan done, carry known, tile done.
__device__ long long g_gae_prof[16384][6];
#define GAE_STAMP(k) \
  if (tid == ((k) == 4 ? kGaeThreads - 32 : 0) && t < 16384) g_gae_prof[t][k] = clock64()
#else
#define GAE_STAMP(k)
#endif

template <bool kBulk>
__global__ void __launch_bounds__(kGaeThreads) gae_pipe_kernel(const GaeArgs g, GaeWs ws) {
  __shared__ GaeStage stg[2];
  __shared__ __align__(8) uint64_t full[2];
  __shared__ uint32_t last_bits[kGaeTile / 32];  // bit j: token lo+j ends a sequence
  __shared__ Aff wtot[kGaeThreads / 32];
  __shared__ double2 carry;
  __shared__ int64_t s_tile[2], s_k[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double gamma = g.gamma, gl = g.gamma * g.lam;
  const int64_t in_lo = __ldg(g.cu), in_hi = min64(g.n_tokens, __ldg(g.cu + g.nseq));
  // a tile goes by bulk copy when it is full (sizes multiple of 16 B)
  auto bulk_ok = [&](int64_t t) { return kBulk && (t + 1) * kGaeTile <= g.n_tokens; };
  auto claim = [&]() { return g.ntiles - 1 - int64_t(atomicAdd(ws.ticket, 1u)); };
  auto issue = [&](int64_t t, int s) {  // thread 0
    const int64_t lo = t * kGaeTile;
    const uint64_t pol = l2_evict_first_policy();
    mbar_arrive_expect_tx(&full[s], (g.mask ? 9u : 8u) * kGaeTile);
    bulk_g2s(stg[s].v, g.values + lo, 4u * kGaeTile, &full[s], pol);
    bulk_g2s(stg[s].r, g.rewards + lo, 4u * kGaeTile, &full[s], pol);
    if (g.mask) bulk_g2s(stg[s].m, g.mask + lo, kGaeTile, &full[s], pol);
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
    const int64_t t0 = claim();
    s_tile[0] = t0;
    if (t0 >= 0 && bulk_ok(t0)) issue(t0, 0);
  }
  __syncthreads();
  int s = 0;
  uint32_t phase[2] = {0u, 0u};
  for (int64_t t = s_tile[0]; t >= 0; t = s_tile[s ^= 1]) {
    if (tid == 0) {  // keep the next tile in flight while this one is scanned
      const int64_t nx = claim();
      s_tile[s ^ 1] = nx;
      if (nx >= 0 && bulk_ok(nx)) issue(nx, s ^ 1);
    }
    GAE_STAMP(0);
    const int64_t lo = t * kGaeTile, hi = min64(g.n_tokens, lo + kGaeTile);
    for (int i = tid; i < kGaeTile / 32; i += kGaeThreads) last_bits[i] = 0u;
    if (warp < 2) {  // sequence ends in the tile: k with cu[k] in [lo+1, hi]
      const int64_t k = warp_lower_bound(g.cu, 1, g.nseq + 1, (warp == 0 ? lo : hi) + 1, lane);
      if (lane == 0) s_k[warp] = k;
    }
    GaeStage& S = stg[s];
    if (bulk_ok(t)) {
      mbar_wait(&full[s], phase[s]);
      phase[s] ^= 1u;
      GAE_STAMP(1);
    } else {  // ragged last tile or unaligned arrays: cooperative element loads
      for (int64_t i = lo + tid; i < lo + kGaeTile; i += kGaeThreads) {
        const bool ok = i < hi;
        S.v[i - lo] = ok ? g.values[i] : 0.f;
        S.r[i - lo] = ok ? g.rewards[i] : 0.f;
        S.m[i - lo] = ok ? (g.mask ? g.mask[i] : uint8_t(1)) : uint8_t(0);
      }
    }
    __syncthreads();
    for (int64_t k = s_k[0] + tid; k < s_k[1]; k += kGaeThreads) {
      const int64_t j = __ldg(g.cu + k) - 1 - lo;
      atomicOr(&last_bits[j >> 5], 1u << (j & 31));
    }
    __syncthreads();
    GAE_STAMP(2);
    const int j0 = tid * kGaeTpt;  // this thread's first token within the tile
    const int64_t x0 = lo + j0;
    const int nmine = int(max64(0, min64(kGaeTpt, hi - x0)));
    // 16-bit masks over this thread's tokens: inside [cu[0], cu[nseq]) and
    // the array, valid (mask != 0), last token of a sequence
    const uint32_t lb = (last_bits[j0 >> 5] >> (j0 & 31)) & 0xffffu;
    uint32_t insm = 0u, validm = 0xffffu;
    {
      const int64_t a = max64(0, in_lo - x0), b = min64(nmine, in_hi - x0);
      if (b > a) insm = ((1u << b) - 1u) & ~((1u << a) - 1u);
    }
    if (g.mask) {
      const uint4 m4 = *reinterpret_cast<const uint4*>(S.m + j0);
      const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
      validm = 0u;
#pragma unroll
      for (int j = 0; j < kGaeTpt; ++j)
        validm |= ((mw[j >> 2] >> (8 * (j & 3))) & 0xffu) ? (1u << j) : 0u;
    }

    // compose this thread's tokens right to left
    Aff f = aff_id();
#pragma unroll
    for (int q = kGaeTpt / 4 - 1; q >= 0; --q) {
      const float4 v4 = *reinterpret_cast<const float4*>(S.v + j0 + 4 * q);
      const float4 r4 = *reinterpret_cast<const float4*>(S.r + j0 + 4 * q);
      const float vq[4] = {v4.x, v4.y, v4.z, v4.w}, rq[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
      for (int u = 3; u >= 0; --u) {
        const uint32_t bit = 1u << (4 * q + u);
        if (!(insm & bit)) continue;
        if (lb & bit) f = Aff{0.0, 0.0, 0.0, 0.0, 0.0};
        if (validm & bit) {
          const double vv = f2d(vq[u]);
          f = Aff{gl * f.a, gl * f.b + gamma * f.k, 0.0,
                  gl * f.p + gamma * f.q + (f2d(rq[u]) - vv), vv};
        }
      }
    }
    // inclusive scan from the right inside the warp, then warp totals
    Aff inc = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const Aff o = shfl_down_aff(inc, d);
      if (lane + d < 32) inc = compose(inc, o);
    }
    if (lane == 0) wtot[warp] = inc;
    __syncthreads();
    GAE_STAMP(3);
    // composite of the threads to my right: later lanes, then later warps
    Aff right = aff_id();
    for (int w = kGaeThreads / 32 - 1; w > warp; --w) right = compose(wtot[w], right);
    Aff ex = shfl_down_aff(inc, 1);
    if (lane == 31) ex = aff_id();
    ex = compose(ex, right);
    // replay right to left from shared memory, four tokens per step
    const bool all_in = insm == 0xffffu;
    auto replay = [&](double A, double Vn) {
#pragma unroll
      for (int q = kGaeTpt / 4 - 1; q >= 0; --q) {
        const float4 v4 = *reinterpret_cast<const float4*>(S.v + j0 + 4 * q);
        const float4 r4 = *reinterpret_cast<const float4*>(S.r + j0 + 4 * q);
        const float vq[4] = {v4.x, v4.y, v4.z, v4.w}, rq[4] = {r4.x, r4.y, r4.z, r4.w};
        float ao[4], ro[4];
#pragma unroll
        for (int u = 3; u >= 0; --u) {
          const uint32_t bit = 1u << (4 * q + u);
          ao[u] = 0.f, ro[u] = 0.f;
          if (!(insm & bit)) continue;
          if (lb & bit) A = 0.0, Vn = 0.0;
          const double vv = f2d(vq[u]);
          if (validm & bit) {
            A = (f2d(rq[u]) - vv) + gamma * Vn + gl * A;
            Vn = vv;
          }
          ao[u] = float(A);
          ro[u] = float(A + vv);
        }
        if (kBulk && all_in) {
          __stcs(reinterpret_cast<float4*>(g.adv + x0) + q, make_float4(ao[0], ao[1], ao[2], ao[3]));
          __stcs(reinterpret_cast<float4*>(g.ret + x0) + q, make_float4(ro[0], ro[1], ro[2], ro[3]));
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (insm & (1u << (4 * q + u))) {
              g.adv[x0 + 4 * q + u] = ao[u];
              g.ret[x0 + 4 * q + u] = ro[u];
            }
        }
      }
    };
    // lane 0 of the last warp publishes the tile and looks back; meanwhile
    // every thread with a sequence end to its right inside the tile (constant
    // right composite) replays without waiting for the carry
    if (tid == kGaeThreads - 32) {
      Aff tot = wtot[kGaeThreads / 32 - 1];
      for (int w = kGaeThreads / 32 - 2; w >= 0; --w) tot = compose(wtot[w], tot);
      const bool constant = tot.a == 0.0 && tot.b == 0.0 && tot.k == 0.0;
      if (constant) {
        st_incl(ws.incl + t, tot.p, tot.q);
      } else {
        ws.agg[t] = tot;
        st_release(ws.aflag + t, 1u);
      }
      // look-back: state entering from the right = M_{t+1} o ... o (state of
      // the first tile to the right that published its outgoing state)
      Aff c = aff_id();
      double2 st = make_double2(0.0, 0.0);
      for (int64_t j = t + 1; j < g.ntiles; ++j) {
        int spins = 0;
        for (;;) {
          const uint4 w = ld_incl(ws.incl + j);
          if (w.w != 0u) {
            st = make_double2(__hiloint2double(int(w.y), int(w.x)), double(__uint_as_float(w.z)));
            j = g.ntiles;  // done
            break;
          }
          if (ld_acquire(ws.aflag + j) != 0u) {
            const Aff* a = ws.agg + j;
            c = compose(c, Aff{__ldcg(&a->a), __ldcg(&a->b), __ldcg(&a->k), __ldcg(&a->p),
                               __ldcg(&a->q)});
            break;
          }
          if (++spins > 4) __nanosleep(32);
        }
      }
      const double2 in_state = make_double2(c.a * st.x + c.b * st.y + c.p, c.k * st.y + c.q);
      if (!constant)
        st_incl(ws.incl + t, tot.a * in_state.x + tot.b * in_state.y + tot.p,
                tot.k * in_state.y + tot.q);
      carry = in_state;
      GAE_STAMP(4);
    }
    const bool need_carry = !(ex.a == 0.0 && ex.b == 0.0 && ex.k == 0.0);
    if (!need_carry) replay(ex.p, ex.q);
    __syncthreads();
    if (need_carry) {
      const double2 cs = carry;
      replay(ex.a * cs.x + ex.b * cs.y + ex.p, ex.k * cs.y + ex.q);
    }
    __syncthreads();  // stage s, last_bits, wtot and carry are reused next
    GAE_STAMP(5);
  }
}

int gae_pipe_occupancy(bool bulk) {
  static int occ[2] = {0, 0};
  int& o = occ[bulk ? 1 : 0];
  if (o == 0) {
    int n = 0;
    if (bulk)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gae_pipe_kernel<true>, kGaeThreads, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, gae_pipe_kernel<false>, kGaeThreads, 0);
    o = n > 0 ? n : 1;
  }
  return o;
}

// ------------------------------------------------------- masked moments ----
constexpr int kMomThreads = 256;
constexpr int kMomMaxParts = 640;

__device__ __forceinline__ void mom_add(float x, bool valid, double& c, double& s, double& q) {
  if (valid) {
    const double v = f2d(x);
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
  double v = (f2d(x) - w.mean) * w.inv;
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
  return gae_ws_bytes(ceil_div(max64(n_tokens, 0), kGaeTile));
}

int gae_launch(const float* values, const float* rewards, const uint8_t* mask, const int64_t* cu,
               int64_t nseq, int64_t n_tokens, float gamma, float lam, float* adv, float* ret,
               void* ws, size_t ws_bytes, cudaStream_t st) {
  YATT_REQUIRE(nseq >= 0 && n_tokens >= 0, YATT_ERR_CONFIG, "gae: n_seqs and n_tokens must be >= 0");
  YATT_REQUIRE(gamma >= 0.f && lam >= 0.f, YATT_ERR_CONFIG, "gae: gamma/lam must be >= 0");
  if (nseq == 0 || n_tokens == 0) return YATT_OK;
  YATT_REQUIRE(values && rewards && cu && adv && ret, YATT_ERR_CONFIG, "gae: null pointer");
  const int64_t ntiles = ceil_div(n_tokens, kGaeTile);
  YATT_REQUIRE(ws != nullptr && ws_bytes >= gae_ws_bytes(ntiles), YATT_ERR_WORKSPACE,
               "gae: workspace too small (%zu < %zu)", ws_bytes, gae_ws_bytes(ntiles));
  YATT_REQUIRE(ntiles < (int64_t(1) << 31), YATT_ERR_CONFIG, "gae: too many tokens");
  YATT_TRY_CUDA(cudaMemsetAsync(ws, 0, gae_zero_bytes(ntiles), st));
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool bulk = a16(values) && a16(rewards) && a16(mask) && a16(adv) && a16(ret);
  const GaeArgs args{values, rewards, mask, cu, nseq, n_tokens, ntiles, double(gamma), double(lam),
                     adv, ret};
  const int grid = int(min64(ntiles, int64_t(num_sms()) * gae_pipe_occupancy(bulk)));
  if (bulk)
    gae_pipe_kernel<true><<<grid, kGaeThreads, 0, st>>>(args, gae_ws(ws, ntiles));
  else
    gae_pipe_kernel<false><<<grid, kGaeThreads, 0, st>>>(args, gae_ws(ws, ntiles));
  return check_launch("gae_pipe_kernel");
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
