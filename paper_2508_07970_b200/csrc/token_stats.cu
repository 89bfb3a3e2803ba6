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
#include "online_lse.cuh"

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
static_assert(kVecPerTile % kConsumers == 0, "tile must split evenly");

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

#ifndef YATT_A1_SMALL_TU
// ----------------------------------------------------------------------
// Small vocabularies: one WARP per row.  With short rows the ring kernel's
// per-row cost (a CTA-wide barrier after the thread -> warp combine, then a
// rotating warp's fp64 epilogue) is a large share of a row: at V = 8,192 it
// ran at 0.55-0.61 of the HBM peak.  Here every warp owns whole rows: its
// lane 0 streams the warp's rows in 1,024-logit chunks of both tensors into
// the warp's own 2-stage shared-memory ring (cp.async.bulk, an mbarrier per
// stage), the lanes fold each chunk into their accumulators with a per-chunk
// max + exact rebase (no overflow, no fix-up pass), and the row end is a warp
// shuffle combine plus lane 0's fp64 epilogue — no CTA barrier, and while a
// warp is at its row end its next chunks keep loading.  2 CTAs x 8 warps per
// SM (1 x 8 with 4 stages: 0.73 at V = 8,192, 3 x 8: spills).  V % 8 == 0,
// 16-byte-aligned tensors.
#ifndef YATT_A1_RW_MINB
#define YATT_A1_RW_MINB 2
#endif
#ifndef YATT_A1_RW_STAGES
#define YATT_A1_RW_STAGES 2
#endif
constexpr int kRWWarps = 8;                    // warps per CTA
constexpr int kRWMinB = YATT_A1_RW_MINB;       // CTAs per SM
constexpr int kRWChunk = 1024;                 // logits per tensor per chunk
constexpr int kRWStages = YATT_A1_RW_STAGES;   // chunks in flight per warp
constexpr int kRWVec = kRWChunk / 8 / 32;      // 16-byte vectors per lane per tensor
constexpr size_t kRWStageBytes = size_t(2) * kRWChunk * sizeof(uint16_t);  // pol + ref
constexpr size_t kRWWarpBytes = kRWStages * kRWStageBytes + kRWStages * sizeof(uint64_t);
constexpr size_t kRWSmem = kRWWarps * kRWWarpBytes;
static_assert(kRWVec * 8 * 32 == kRWChunk, "row-warp chunk");

template <bool kFull>
__global__ void __launch_bounds__(kRWWarps * 32, kRWMinB) token_stats_rowwarp_kernel(
    const A1Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbase = smem + size_t(warp) * kRWStages * kRWStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRWWarps * kRWStages * kRWStageBytes) +
                   warp * kRWStages;
  const int V = int(p.V);
  const int nch = (V + kRWChunk - 1) / kRWChunk;
  const int64_t gw = int64_t(blockIdx.x) * kRWWarps + warp, nw = int64_t(gridDim.x) * kRWWarps;
  if (lane == 0) {
    for (int s = 0; s < kRWStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // The warp's chunk stream: (row, chunk) for its valid rows, in order.
  // Lane 0 keeps kRWStages chunks in flight ahead of the consumer.
  const uint64_t pol_hint = l2_evict_first_policy();
  int64_t prow = gw;  // producer cursor
  int pch = 0;
  auto next_valid = [&](int64_t r) {
    while (r < p.rows && p.mask != nullptr && p.mask[r] == 0) r += nw;
    return r;
  };
  auto issue = [&](int slot) {  // lane 0: the next chunk of the stream into `slot`
    if (prow >= p.rows) return;
    const int e0 = pch * kRWChunk;
    const uint32_t n = uint32_t(min(kRWChunk, V - e0));
    uint16_t* dst = reinterpret_cast<uint16_t*>(wbase + size_t(slot) * kRWStageBytes);
    mbar_arrive_expect_tx(&full[slot], 4u * n);
    bulk_g2s(dst, p.pol + prow * int64_t(V) + e0, 2u * n, &full[slot], pol_hint);
    bulk_g2s(dst + kRWChunk, p.ref + prow * int64_t(V) + e0, 2u * n, &full[slot], pol_hint);
    if (++pch == nch) {
      pch = 0;
      prow = next_valid(prow + nw);
    }
  };
  if (lane == 0) {
    prow = next_valid(prow);
    for (int s = 0; s < kRWStages; ++s) issue(s);
  }
  int slot = 0;
  uint32_t phase = 0;
  Acc<kFull> acc;
  for (int64_t row = gw; row < p.rows; row += nw) {
    if (p.mask != nullptr && p.mask[row] == 0) {
      if (lane == 0) {
        p.logp[row] = 0.f;
        if (p.ref_logp) p.ref_logp[row] = 0.f;
        if (p.ent) p.ent[row] = 0.f;
        if (p.kl) p.kl[row] = 0.f;
      }
      continue;
    }
    const int32_t y = __ldg(p.tgt + row);
    const bool yok = y >= 0 && y < V;
    const int yc = yok ? y / kRWChunk : -1, yin = yok ? y - yc * kRWChunk : 0;
    const int ylane = (yin >> 3) & 31;
    float xy = 0.f, zy = 0.f;
    acc.reset();
    for (int c = 0; c < nch; ++c) {
      const uint16_t* sp = reinterpret_cast<const uint16_t*>(wbase + size_t(slot) * kRWStageBytes);
      const uint16_t* sq = sp + kRWChunk;
      const int nvec = min(kRWChunk, V - c * kRWChunk) >> 3;
      mbar_wait(&full[slot], phase);
      if (c == yc && lane == ylane) {
        xy = __uint_as_float(uint32_t(sp[yin]) << 16);
        zy = __uint_as_float(uint32_t(sq[yin]) << 16);
      }
      uint4 P[kRWVec], Q[kRWVec];
      const uint4 ninf = make_uint4(kNegInf2, kNegInf2, kNegInf2, kNegInf2);
#pragma unroll
      for (int i = 0; i < kRWVec; ++i) {
        const int v = lane + 32 * i;
        const bool in = nvec == kRWChunk / 8 || v < nvec;
        P[i] = floor_policy(in ? lds128(sp + v * 8) : ninf);
        Q[i] = in ? lds128(sq + v * 8) : ninf;
        if (kFull) Q[i] = floor_policy(Q[i]);
      }
      uint32_t mpv = vmax4(P[0]), mqv = vmax4(Q[0]);
#pragma unroll
      for (int i = 1; i < kRWVec; ++i) {
        mpv = bmax2(mpv, vmax4(P[i]));
        mqv = bmax2(mqv, vmax4(Q[i]));
      }
      const float fmp = pair_max(mpv), fmq = pair_max(mqv);
      if (fmp > acc.thr_p) acc.rebase_p(fmp);
      if (fmq > acc.thr_q) acc.rebase_q(fmq);
#pragma unroll
      for (int i = 0; i < kRWVec; ++i) acc.step(P[i], Q[i]);
      __syncwarp();  // every lane's reads of the slot are done: refill it
      if (lane == 0) issue(slot);
      if (++slot == kRWStages) {
        slot = 0;
        phase ^= 1u;
      }
    }
    RowPartial r{acc.mp, Acc<kFull>::total(acc.s), Acc<kFull>::total(acc.w), acc.mq,
                 Acc<kFull>::total(acc.sq), kFull ? Acc<kFull>::total(acc.u) : 0.f};
    r = warp_combine<kFull>(r);
    xy = __shfl_sync(0xffffffffu, xy, ylane);
    zy = __shfl_sync(0xffffffffu, zy, ylane);
    if (lane == 0) {
      const float nan = __uint_as_float(0x7fc00000u);
      emit_row(p, row, r, yok ? xy : nan, yok ? zy : nan);
    }
  }
}
#endif  // !YATT_A1_SMALL_TU

}  // namespace

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


#ifndef YATT_A1_SMALL_TU
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
// Vocabularies up to this (V % 8 == 0) take the warp-per-row kernel.
// Fraction of the measured HBM peak, warp-per-row vs ring (k3 / full KL,
// profiles/r2_a1_rowwarp_v*.jsonl): V=8,192 0.911 vs 0.611 / 0.860 vs 0.576;
// 24,576 0.959 vs 0.887 / 0.934 vs 0.819; 32,000 0.942 vs 0.903 / 0.898 vs
// 0.832; 40,960 0.924 vs 0.934 / 0.890 vs 0.892; 65,536 0.869 vs 0.957.
// YATT_A1_ROWWARP_VMAX overrides (measurement only).
int a1_rowwarp_vmax() {
  const char* e = std::getenv("YATT_A1_ROWWARP_VMAX");
  return e ? std::atoi(e) : 36864;
}

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
  if (vocab % 8 == 0 && vocab <= a1_rowwarp_vmax()) {
    const void* k = kl_mode == YATT_KL_FULL
                        ? reinterpret_cast<const void*>(token_stats_rowwarp_kernel<true>)
                        : reinterpret_cast<const void*>(token_stats_rowwarp_kernel<false>);
    const int rc = ensure_dynamic_smem(k, int(kRWSmem));
    if (rc) return rc;
    const int grid = int(min64(ceil_div(rows, kRWWarps), int64_t(kRWMinB) * num_sms()));
    if (kl_mode == YATT_KL_FULL)
      token_stats_rowwarp_kernel<true><<<grid, kRWWarps * 32, kRWSmem, st>>>(p);
    else
      token_stats_rowwarp_kernel<false><<<grid, kRWWarps * 32, kRWSmem, st>>>(p);
    return check_launch("token_stats_rowwarp_kernel");
  }
  return vocab <= a1_small_vmax() ? token_stats_ring_small(p, st) : token_stats_ring_large(p, st);
}
#endif  // !YATT_A1_SMALL_TU

}  // namespace yattb
