// lmhead_lse.cu — §8f #4: fused LM-head GEMM + online log-softmax on tcgen05.
//
// The step before A1 (Stage 3: "the policy and reference policy
// compute their reference log probabilities"; stand-in simcore.cpp:13-15):
// logits = hidden[rows, d] · W[V, d]^T are never written to HBM — each 128 x
// 256 accumulator tile goes TMEM -> registers -> an online log-sum-exp /
// entropy update, and only per-row (lse, logp, entropy) leave the SM.
//
//   warp 0      TMA producer: 2-D tensor-map loads (128-B swizzle) of a
//               128 x 64 hidden tile and a 256 x 64 weight tile per stage into
//               a 4-stage shared-memory ring (mbarrier transaction counts)
//   warp 1      allocates 512 TMEM columns; one elected thread issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16, bf16 ->
//               fp32) from smem descriptors, tcgen05.commit frees ring stages
//               and hands finished accumulators to the epilogue
//   warps 2..5  epilogue: tcgen05.ld.32x32b.x32 (one thread = one row), online
//               log2-domain LSE with integer bases + entropy accumulator, packed
//               f32x2 math; double-buffered accumulators (2 x 256 columns) let
//               tile j+1's MMAs run under tile j's epilogue
// Grid: (row tiles, vocabulary splits); lmhead_combine merges the splits'
// (m, s, w) partials, adds the target logit (fp32 dot product) and emits
// logp / entropy / lse.  FLOPs per token = 2 d V (tensor bound).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace yattb {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, UMMA_K = 16;
constexpr int kStagesG = 4;
constexpr int kABytes = BM * BK * 2;  // 16 KB
constexpr int kBBytes = BN * BK * 2;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kGemmThreads = 192;  // 6 warps
constexpr int kTmemCols = 512;
constexpr float kL2e = 1.4426950408889634f;

struct __align__(8) GemmBars {
  uint64_t full[kStagesG];
  uint64_t empty[kStagesG];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};
constexpr size_t kGemmSmem = size_t(kStagesG) * kStageBytes + 1024 /*align*/ + sizeof(GemmBars);

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// K-major operand, 128-byte swizzle: rows of 64 bf16 (128 B), 8-row atoms of
// 1024 B (stride byte offset), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D, K-major A and B.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define TMEM_LD32(taddr, r)                                                                      \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"         \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),     \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),           \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),           \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])            \
      : "r"(taddr))

struct LseState {
  float m;        // integer base (log2 units)
  double s, w;    // sum 2^a, sum 2^a * a (fp64 across the ~5K chunks of a row)
};

// Online log2 LSE + entropy over one BN-column accumulator tile: this
// thread's row, columns [n0, min(n0 + BN, v1)) read from TMEM 32 at a time.
__device__ __forceinline__ void lse_tile(uint32_t tbase, int n0, int v1, LseState& st) {
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t r[32];
    TMEM_LD32(tbase + uint32_t(c * 32), r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int colbase = n0 + c * 32;
    const int valid = min(32, v1 - colbase);  // partial last tile
    float cmax = -INFINITY;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < valid) cmax = fmaxf(cmax, __uint_as_float(r[k]));
    if (valid > 0 && cmax * kL2e > st.m + 24.f) {  // rebase (exact power of two)
      const float mn = ceilf(cmax * kL2e);
      const double dd = double(st.m) - double(mn);
      const double cs = exp2(fmax(dd, -1000.0));
      st.w = cs * (dd * st.s + st.w);
      st.s *= cs;
      st.m = mn;
    }
    float2 s2 = make_float2(0.f, 0.f), w2 = s2;
    const float2 L2 = make_float2(kL2e, kL2e), nm = make_float2(-st.m, -st.m);
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      const float2 x = make_float2(k < valid ? __uint_as_float(r[k]) : -INFINITY,
                                   k + 1 < valid ? __uint_as_float(r[k + 1]) : -INFINITY);
      float2 a = __ffma2_rn(x, L2, nm);
      a = make_float2(fmaxf(a.x, -200.f), fmaxf(a.y, -200.f));  // masked cols -> 0
      const float2 e = make_float2(ex2_approx(a.x), ex2_approx(a.y));
      s2 = __fadd2_rn(s2, e);
      w2 = __ffma2_rn(e, a, w2);
    }
    st.s += double(s2.x + s2.y);
    st.w += double(w2.x + w2.y);
  }
}

__device__ __forceinline__ void tma_load_2d_mcast(void* dst, const CUtensorMap* map, int x, int y,
                                                  uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mcast(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// kCluster = 2: CTA pairs on adjacent row tiles (cluster dims 1x2) share the
// weight tile: each loads its own hidden tile and HALF of the weight tile,
// multicast into both CTAs' shared memory (a third less L2->SM traffic per
// CTA); a ring stage is reused only after BOTH CTAs' MMAs retired it
// (multicast tcgen05.commit, empty barriers count 2).
// Work units (row tile, vocabulary split), split fastest.  A launch either
// maps one unit per CTA (grid = units, the first waves' tail idles SMs) or
// runs persistent CTAs (grid = SMs) that walk the units in the same order
// with their ring / accumulator pipelines continuing across units.
template <int kCluster>
__global__ void __launch_bounds__(kGemmThreads, 1) lmhead_lse_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    int64_t rows, int32_t V, int32_t d, int32_t v_per_split, int32_t nsplit, int64_t nunits,
    float4* partial) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  GemmBars* bars = reinterpret_cast<GemmBars*>(smem + size_t(kStagesG) * kStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Rasterisation: vocabulary split fastest, so the CTAs resident at one time
  // cover few row tiles (their hidden tiles stay in L2) and walk the same
  // weight tiles together.
  const int64_t u_first = int64_t(blockIdx.y) * gridDim.x + blockIdx.x;
  const int64_t u_stride = int64_t(gridDim.x) * gridDim.y;
  const int nk = (d + BK - 1) / BK;
  struct Unit {
    int64_t m0;
    int v0, v1, ntiles;
  };
  auto unit = [&](int64_t u) {
    Unit x;
    x.m0 = (u / nsplit) * BM;
    x.v0 = int(u % nsplit) * v_per_split;
    x.v1 = min(V, x.v0 + v_per_split);
    x.ntiles = (x.v1 - x.v0 + BN - 1) / BN;
    return x;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesG; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], kCluster);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bars->tfull[a], 1);
      mbar_init(&bars->tempty[a], 4);
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&bars->tmem_base)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (kCluster > 1) cluster_sync_all();  // peer barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const uint32_t crank = kCluster > 1 ? cluster_rank() : 0u;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer ----
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = u_first; u < nunits; u += u_stride) {
      const Unit w = unit(u);
      const int64_t m0 = w.m0;
      for (int j = 0; j < w.ntiles; ++j) {
        const int n0 = w.v0 + j * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&bars->empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx(&bars->full[stage], kStageBytes);
          uint8_t* sa = smem + size_t(stage) * kStageBytes;
          tma_load_2d(sa, &tmA, kb * BK, int(m0), &bars->full[stage]);
          if (kCluster > 1)  // my half of the weight tile, into both CTAs
            tma_load_2d_mcast(sa + kABytes + crank * (kBBytes / 2), &tmB, kb * BK,
                              n0 + int(crank) * (BN / 2), &bars->full[stage], uint16_t(0x3));
          else
            tma_load_2d(sa + kABytes, &tmB, kb * BK, n0, &bars->full[stage]);
          if (++stage == kStagesG) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      int stage = 0;
      uint32_t phase = 0;
      int jg = 0;  // accumulator tiles so far (across units)
      for (int64_t u = u_first; u < nunits; u += u_stride) {
      const Unit w = unit(u);
      for (int j = 0; j < w.ntiles; ++j, ++jg) {
        const int acc = jg & 1;
        const uint32_t aphase = (jg >> 1) & 1;
        mbar_wait(&bars->tempty[acc], aphase ^ 1u);
        tc_fence_after();
        const uint32_t tmem_d = tmem + uint32_t(acc * BN);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&bars->full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + size_t(stage) * kStageBytes);
          const uint64_t adesc = sdesc_sw128(sa), bdesc = sdesc_sw128(sa + kABytes);
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            // +32 bytes along K inside the 128-B swizzle atom = +2 in the
            // descriptor's 16-byte address units
            umma(tmem_d, adesc + uint64_t(2 * kk), bdesc + uint64_t(2 * kk),
                 (kb | kk) != 0 ? 1u : 0u);
          }
          if (kCluster > 1)  // stage free once BOTH CTAs' MMAs retired it
            umma_commit_mcast(&bars->empty[stage], uint16_t(0x3));
          else
            umma_commit(&bars->empty[stage]);
          if (++stage == kStagesG) {
            stage = 0;
            phase ^= 1u;
          }
        }
        umma_commit(&bars->tfull[acc]);  // accumulator ready for the epilogue
      }
      }
    }
  } else {
    // ---- epilogue: warps 2..5, TMEM lane quarter = warp % 4 ----
    const int quarter = warp & 3;
    int jg = 0;
    for (int64_t u = u_first; u < nunits; u += u_stride) {
    const Unit w = unit(u);
    const int v1 = w.v1;
    const int64_t row = w.m0 + quarter * 32 + lane;
    LseState st{-float(1 << 24), 0.0, 0.0};
    for (int j = 0; j < w.ntiles; ++j, ++jg) {
      const int acc = jg & 1;
      const uint32_t aphase = (jg >> 1) & 1;
      mbar_wait(&bars->tfull[acc], aphase);
      tc_fence_after();
      const int n0 = w.v0 + j * BN;
      const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
      lse_tile(tbase, n0, v1, st);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->tempty[acc]);
    }
    if (row < rows) {  // normalised so s fits fp32 exactly enough
      const int k = st.s > 0 ? ilogb(st.s) : 0;
      partial[(u % nsplit) * rows + row] =
          make_float4(st.m + float(k), float(ldexp(st.s, -k)), float(ldexp(st.w - k * st.s, -k)), 0.f);
    }
    }
  }
  __syncthreads();
  if (kCluster > 1) cluster_sync_all();  // no remote arrivals/writes pending on exit
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ----------------------------------------------------------------------
// CTA-pair form (cta_group::2): two SMs of one TPC compute a 256 x 256
// accumulator tile together.  Each CTA loads its 128 rows of the hidden
// tile and HALF (128 columns) of the weight tile per K-step (16 + 16 KB, so
// a 6-stage ring); the leader CTA's one thread issues
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16), which reads A from each
// CTA's own shared memory and B from both, and writes each CTA's 128 rows x
// 256 columns into that CTA's TMEM.  Per SM: a third less shared-memory
// operand traffic per FLOP and half the weight bytes from L2.
//   full[s]   leader only: both CTAs' TMA bytes (peer loads signal the
//             leader's barrier: its shared::cluster address with the peer bit
//             cleared), one arrive_expect_tx by the leader
//   empty[s]  each CTA: the leader's MMA commit multicast to both
//   tfull[a]  each CTA: the leader's accumulator commit multicast to both
//   tempty[a] leader only: 4 epilogue warps x 2 CTAs arrive (the peer's
//             remotely) before the accumulator is overwritten
constexpr int kPairStages = 6;
constexpr int kPABytes = BM * BK * 2;           // 16 KB: this CTA's hidden rows
constexpr int kPBBytes = (BN / 2) * BK * 2;     // 16 KB: this CTA's half of the weights
constexpr int kPStageBytes = kPABytes + kPBBytes;
struct __align__(8) PairBars {
  uint64_t full[kPairStages];
  uint64_t empty[kPairStages];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};
constexpr size_t kPairSmem = size_t(kPairStages) * kPStageBytes + 1024 + sizeof(PairBars);
constexpr uint32_t kIdescPair = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                                (uint32_t((2 * BM) >> 4) << 24);
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // shared::cluster address of rank 0's copy

__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescPair), "r"(acc));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(uint16_t(0x3))
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster_acq(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive_cluster_addr(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}

__global__ void __launch_bounds__(kGemmThreads, 1) lmhead_lse_pair_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    int64_t rows, int32_t V, int32_t d, int32_t v_per_split, int32_t nsplit, int64_t nunits,
    float4* partial) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  PairBars* bars = reinterpret_cast<PairBars*>(smem + size_t(kPairStages) * kPStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  // units (row-tile pair, vocabulary split), split fastest; one per cluster
  const int64_t u_first = blockIdx.x >> 1, u_stride = gridDim.x >> 1;
  const int nk = (d + BK - 1) / BK;
  auto unit = [&](int64_t u, int64_t& m0, int& v0, int& v1, int& ntiles) {
    m0 = (u / nsplit) * (2 * BM) + int64_t(rank) * BM;  // this CTA's 128 rows
    v0 = int(u % nsplit) * v_per_split;
    v1 = min(V, v0 + v_per_split);
    ntiles = (v1 - v0 + BN - 1) / BN;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(&bars->full[s], 1);
      mbar_init(&bars->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bars->tfull[a], 1);
      mbar_init(&bars->tempty[a], 8);
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 1) {  // the same warp in both CTAs allocates the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&bars->tmem_base)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs) ----
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = u_first; u < nunits; u += u_stride) {
        int64_t m0;
        int v0, v1, ntiles;
        unit(u, m0, v0, v1, ntiles);
        for (int j = 0; j < ntiles; ++j) {
          const int n0 = v0 + j * BN + int(rank) * (BN / 2);  // this CTA's weight half
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&bars->empty[stage], phase ^ 1u);
            const uint32_t lbar = smem_u32(&bars->full[stage]) & kPeerBitMask;
            if (leader) mbar_arrive_expect_tx(&bars->full[stage], 2u * kPStageBytes);
            const uint32_t sa = smem_u32(smem + size_t(stage) * kPStageBytes);
            tma_load_2d_pair(sa, &tmA, kb * BK, int(m0), lbar);
            tma_load_2d_pair(sa + kPABytes, &tmB, kb * BK, n0, lbar);
            if (++stage == kPairStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---- MMA issuer (leader CTA) ----
      int stage = 0;
      uint32_t phase = 0;
      int jg = 0;
      for (int64_t u = u_first; u < nunits; u += u_stride) {
        int64_t m0;
        int v0, v1, ntiles;
        unit(u, m0, v0, v1, ntiles);
        for (int j = 0; j < ntiles; ++j, ++jg) {
          const int acc = jg & 1;
          const uint32_t aphase = (jg >> 1) & 1;
          mbar_wait_cluster_acq(&bars->tempty[acc], aphase ^ 1u);
          tc_fence_after();
          const uint32_t tmem_d = tmem + uint32_t(acc * BN);
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&bars->full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + size_t(stage) * kPStageBytes);
            const uint64_t adesc = sdesc_sw128(sa), bdesc = sdesc_sw128(sa + kPABytes);
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; ++kk)
              umma_pair(tmem_d, adesc + uint64_t(2 * kk), bdesc + uint64_t(2 * kk),
                        (kb | kk) != 0 ? 1u : 0u);
            umma_commit_pair(&bars->empty[stage]);  // the stage is free in both CTAs
            if (++stage == kPairStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          umma_commit_pair(&bars->tfull[acc]);  // both CTAs' accumulators ready
        }
      }
    }
  } else {
    // ---- epilogue: warps 2..5 of both CTAs, TMEM lane quarter = warp % 4 ----
    const int quarter = warp & 3;
    int jg = 0;
    for (int64_t u = u_first; u < nunits; u += u_stride) {
      int64_t m0;
      int v0, v1, ntiles;
      unit(u, m0, v0, v1, ntiles);
      const int64_t row = m0 + quarter * 32 + lane;
      LseState st{-float(1 << 24), 0.0, 0.0};
      for (int j = 0; j < ntiles; ++j, ++jg) {
        const int acc = jg & 1;
        const uint32_t aphase = (jg >> 1) & 1;
        mbar_wait(&bars->tfull[acc], aphase);
        tc_fence_after();
        const uint32_t tbase = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
        lse_tile(tbase, v0 + j * BN, v1, st);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_addr(mapa_u32(smem_u32(&bars->tempty[acc]), 0u));
      }
      if (row < rows) {
        const int k = st.s > 0 ? ilogb(st.s) : 0;
        partial[(u % nsplit) * rows + row] = make_float4(
            st.m + float(k), float(ldexp(st.s, -k)), float(ldexp(st.w - k * st.s, -k)), 0.f);
      }
    }
  }
  __syncthreads();
  cluster_sync_all();  // no MMA / remote arrival pending on either CTA
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// Merge the vocabulary splits of each row, add the target logit (warp dot
// product in fp32 over d) and write logp / entropy / lse.
__global__ void lmhead_combine_kernel(const float4* partial, int32_t nsplit, int64_t rows,
                                      const uint16_t* hidden, const uint16_t* W, int32_t d,
                                      const int32_t* tgt, float* logp, float* ent, float* lse) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int32_t y = tgt[row];
  const uint16_t* h = hidden + row * int64_t(d);
  const uint16_t* wy = W + int64_t(y) * d;
  float dot = 0.f;
  for (int k = lane * 2; k < d; k += 64) {
    const uint32_t hv = *reinterpret_cast<const uint32_t*>(h + k);
    const uint32_t wv = *reinterpret_cast<const uint32_t*>(wy + k);
    dot = fmaf(bf16_lo(hv), bf16_lo(wv), dot);
    dot = fmaf(bf16_hi(hv), bf16_hi(wv), dot);
  }
  dot = warp_sum(dot);
  if (lane != 0) return;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, partial[s * rows + row].x);
  double S = 0, Wt = 0;
  for (int s = 0; s < nsplit; ++s) {
    const float4 p = partial[s * rows + row];
    const double c = exp2(double(p.x) - double(M));
    S += c * double(p.y);
    Wt += c * (double(p.z) + (double(p.x) - double(M)) * double(p.y));
  }
  const double kLn2 = 0.69314718055994530942;
  const double l = kLn2 * (double(M) + log2(S));
  if (lse) lse[row] = float(l);
  logp[row] = float(double(dot) - l);
  if (ent) ent[row] = float(kLn2 * (log2(S) - Wt / S));
}

__global__ void kl_from_logps_kernel(const float* logp, const float* ref_logp, int64_t n,
                                     int32_t mode, float* kl) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = double(ref_logp[i]) - double(logp[i]);
  kl[i] = float(mode == YATT_KL_K1 ? -d : mode == YATT_KL_K2 ? 0.5 * d * d : expm1(d) - d);
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_map(CUtensorMap* map, const void* base, int64_t rows, int32_t d, int box_rows) {
  static EncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    YATT_TRY_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    YATT_REQUIRE(fn != nullptr && q == cudaDriverEntryPointSuccess, YATT_ERR_CUDA,
                 "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeTiled>(fn);
  }
  const cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(d) * 2};
  const cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  YATT_REQUIRE(r == CUDA_SUCCESS, YATT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return YATT_OK;
}

}  // namespace

// n_split = 0: the library picks — few splits keep the weight stream shared
// in L2, enough to fill the SMs when rows are few (tools/lmhead_sweep.py).
int32_t lmhead_auto_split(int64_t rows, int32_t nsplit) {
  if (nsplit != 0) return nsplit;
  const int64_t tiles = ceil_div(rows > 0 ? rows : 1, BM);
  return int32_t(min64(64, max64(2, num_sms() / tiles)));
}

size_t lmhead_workspace_bytes(int64_t rows, int32_t V, int32_t nsplit) {
  nsplit = lmhead_auto_split(rows, nsplit);
  (void)V;
  return size_t(rows) * size_t(nsplit > 0 ? nsplit : 1) * sizeof(float4);
}

int lmhead_token_stats_launch(const uint16_t* hidden, const uint16_t* W, const int32_t* tgt,
                              int64_t rows, int32_t d, int32_t V, int32_t nsplit, float* logp,
                              float* ent, float* lse, void* ws, size_t ws_bytes,
                              cudaStream_t st) {
  YATT_REQUIRE(rows >= 0 && d > 0 && V > 0, YATT_ERR_CONFIG, "lmhead: bad sizes");
  YATT_REQUIRE(d % 8 == 0, YATT_ERR_CONFIG, "lmhead: hidden size must be a multiple of 8");
  nsplit = lmhead_auto_split(rows, nsplit);
  YATT_REQUIRE(nsplit >= 1 && nsplit <= 64, YATT_ERR_CONFIG, "lmhead: nsplit in [0, 64]");
  if (rows == 0) return YATT_OK;
  YATT_REQUIRE(hidden && W && tgt && logp, YATT_ERR_CONFIG, "lmhead: null pointer");
  YATT_REQUIRE(ws && ws_bytes >= lmhead_workspace_bytes(rows, V, nsplit), YATT_ERR_WORKSPACE,
               "lmhead: workspace too small");
  YATT_REQUIRE((reinterpret_cast<uintptr_t>(hidden) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(W) & 15) == 0,
               YATT_ERR_CONFIG, "lmhead: operands must be 16-byte aligned");
  // The multicast pair (YATT_LMHEAD_CLUSTER=2; round 1): the 1-CTA kernel
  // is already tensor-bound (93% pipe active) after the split-fastest
  // rasterisation and multicasting adds lock-step coupling (1,261 vs 1,296
  // TFLOP/s at 32K rows), so it stays opt-in.
  // Default: the cta_group::2 CTA-pair kernel.  YATT_LMHEAD_CLUSTER = 1 (the
  // single-CTA kernel) or 2 (single-CTA MMAs, weight tiles multicast over a
  // CTA pair) select the alternatives (measurement).  Pair vs single CTA
  // (TFLOP/s, 2 splits; profiles/r2_lmhead_pair_v1.txt): 8K rows x d=3,584 x
  // V=152,064 1,534 vs 1,412; 16K rows 1,302 vs 1,179; 32K rows 1,275 vs
  // 1,223; d=8,192 x V=128,256 1,081 vs 1,111; 4K rows x V=32,000 (4
  // splits) 1,442 vs 1,360 — results bit-identical.
  const char* ce = getenv("YATT_LMHEAD_CLUSTER");
  const bool pair = !(ce && (ce[0] == '1' || ce[0] == '2'));
  const int cluster = (ce && ce[0] == '2') ? 2 : 1;
  CUtensorMap ta, tb;
  int rc = make_map(&ta, hidden, rows, d, BM);
  if (!rc) rc = make_map(&tb, W, V, d, (cluster == 2 || pair) ? BN / 2 : BN);
  if (rc) return rc;
  int v_per_split = int(ceil_div(ceil_div(V, nsplit), BN) * BN);
  const int nsplit_eff = int(ceil_div(V, v_per_split));
  float4* partial = static_cast<float4*>(ws);
  if (pair) {
    const void* k = reinterpret_cast<const void*>(lmhead_lse_pair_kernel);
    rc = ensure_dynamic_smem(k, int(kPairSmem));
    if (rc) return rc;
    const int64_t units = ceil_div(rows, 2 * BM) * nsplit_eff;
    // YATT_LMHEAD_PERSIST=1: one cluster per SM pair walking the units
    const char* pe = getenv("YATT_LMHEAD_PERSIST");
    const int64_t clusters = (pe && pe[0] == '1') ? min64(units, num_sms() / 2) : units;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(unsigned(2 * clusters));
    lc.blockDim = dim3(kGemmThreads);
    lc.dynamicSmemBytes = kPairSmem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    YATT_TRY_CUDA(cudaLaunchKernelEx(&lc, lmhead_lse_pair_kernel, ta, tb, rows, V, d, v_per_split,
                                     int32_t(nsplit_eff), units, partial));
    rc = check_launch("lmhead_lse_pair_kernel");
    if (rc) return rc;
    lmhead_combine_kernel<<<unsigned(ceil_div(rows * 32, 256)), 256, 0, st>>>(
        partial, nsplit_eff, rows, hidden, W, d, tgt, logp, ent, lse);
    return check_launch("lmhead_combine_kernel");
  }
  rc = ensure_dynamic_smem(reinterpret_cast<const void*>(lmhead_lse_kernel<1>), int(kGemmSmem));
  if (!rc) rc = ensure_dynamic_smem(reinterpret_cast<const void*>(lmhead_lse_kernel<2>), int(kGemmSmem));
  if (rc) return rc;
  const int64_t mtiles = ceil_div(ceil_div(rows, BM), cluster) * cluster;
  YATT_REQUIRE(mtiles <= 65535, YATT_ERR_CONFIG, "lmhead: too many rows per launch");
  const int64_t nunits = mtiles * nsplit_eff;
  // YATT_LMHEAD_PERSIST=1: one persistent CTA per SM walking the units
  // (measurement only)
  const char* pe = getenv("YATT_LMHEAD_PERSIST");
  const bool persist = cluster == 1 && pe && pe[0] == '1';
  const dim3 grid = persist ? dim3(unsigned(min64(nunits, num_sms())), 1u, 1u)
                            : dim3(unsigned(nsplit_eff), unsigned(mtiles), 1u);
  if (cluster == 2) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(kGemmThreads);
    lc.dynamicSmemBytes = kGemmSmem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 2;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    YATT_TRY_CUDA(cudaLaunchKernelEx(&lc, lmhead_lse_kernel<2>, ta, tb, rows, V, d, v_per_split,
                                     int32_t(nsplit_eff), nunits, partial));
  } else {
    lmhead_lse_kernel<1><<<grid, kGemmThreads, kGemmSmem, st>>>(
        ta, tb, rows, V, d, v_per_split, int32_t(nsplit_eff), nunits, partial);
  }
  rc = check_launch("lmhead_lse_kernel");
  if (rc) return rc;
  lmhead_combine_kernel<<<unsigned(ceil_div(rows * 32, 256)), 256, 0, st>>>(
      partial, nsplit_eff, rows, hidden, W, d, tgt, logp, ent, lse);
  return check_launch("lmhead_combine_kernel");
}

int kl_from_logps_launch(const float* logp, const float* ref_logp, int64_t n, int32_t mode,
                         float* kl, cudaStream_t st) {
  YATT_REQUIRE(mode >= YATT_KL_K1 && mode <= YATT_KL_K3, YATT_ERR_CONFIG,
               "kl_from_logps: mode must be k1, k2 or k3");
  if (n <= 0) return YATT_OK;
  kl_from_logps_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(logp, ref_logp, n, mode, kl);
  return check_launch("kl_from_logps_kernel");
}

}  // namespace yattb
