// rollout_rounds.cu — the whole dynamic-sampling round loop of one step on the
// device: every round of every controller shard in ONE persistent kernel.
//
// Replaces the loop of run_rlhf_step (proj/src/simcore.cpp:470-490: per round,
// shard_round_output :157-214 for each shard, then StepAssembler::feed_round's
// continue test :304-311, :382) and, with a round limit of 1, a single
// shard_round_output call.  Semantics per round are those of shard_round.cu
// (keyed draw + rejection per pending sample, pending samples ordered by
// sample index within their shard, microbatches of that order, forced
// acceptance at max_rounds); the round loop's continue decision (sum of
// pending > 0) is taken on the device, so the host sees the device once per
// call, not once per round.
//
// Key observation: whether a pending sample is accepted in a round depends
// only on its id and the round (the keyed rejection test, simcore.cpp:187-198,
// never looks at the drawn lengths), so each sample's whole trajectory is
// known up front.  Kernel: a cooperative grid (every CTA resident), 256-sample
// tiles, TWO grid barriers per launch however many rounds it runs:
//   phase 1  per sample: its fate (acceptance round, forced or not, or still
//            pending after the launch's rounds); per tile and round: the
//            pending count at the round's start; the number of rounds
//            needed (atomic max); all rounds' report / microbatch slots zeroed
//   barrier
//   phase 2  per tile, every round back to back: base = pending count of the
//            shard's earlier tiles, in-tile order by ballot; keyed length
//            draw; a segmented warp reduction over the microbatches of the
//            tile's pending run and one thread per tile issue the integer
//            atomics (exact, order-free)
//   barrier
//   results (final state of the samples, reports, occupied microbatch slots)
//   are stored straight into mapped pinned host memory; the host compacts the
//   slots into the (round, shard, mb_index) list while it builds the reports.
// A call is: one launch (phase 1 reads the packed input in place from the
// mapped stage; YATT_ROUNDS_ZC=0 restores one H2D DMA first), one synchronize.
//
// Normal / LogNormal draws that are not certified equal to glibc
// (keyed_draw.cuh) are logged; the host recomputes exactly those with glibc
// and re-runs the call with them as overrides, so results are bit-exact with
// the reference by construction.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "keyed_draw.cuh"

namespace yattb {

// ---- host glibc draw + certification band --------------------------------
namespace {
double g_tie_band = kDefaultTieBand;

double normal_from_key_glibc(uint64_t key) {
  const double u1 = uniform_from_key(key);
  const double u2 = uniform_from_key(splitmix64(key ^ 0x5bf0a8b1457e1d23ULL));
  return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(kTwoPi * u2);
}
}  // namespace

double tie_band() { return g_tie_band; }

int length_keyed_glibc(const yatt_length_dist& d, uint64_t seed, uint64_t stream, uint64_t step,
                       uint64_t round, uint64_t id) {
  const uint64_t key = hash5(seed, stream, step, round, id);
  switch (d.kind) {
    case YATT_DIST_CONSTANT: return clamp_length(d.p1, d.max_len_tokens);
    case YATT_DIST_UNIFORM: {
      const long long lo = std::llround(d.p1), hi = std::llround(d.p2);
      const double span = static_cast<double>(static_cast<uint64_t>(hi - lo) + 1);
      return clamp_length(static_cast<double>(lo + static_cast<long long>(uniform_from_key(key) * span)),
                          d.max_len_tokens);
    }
    case YATT_DIST_NORMAL: return clamp_length(d.p1 + d.p2 * normal_from_key_glibc(key), d.max_len_tokens);
    default: return clamp_length(std::exp(d.p1 + d.p2 * normal_from_key_glibc(key)), d.max_len_tokens);
  }
}


namespace {

constexpr int kTile = 256;
constexpr int kRoundsPerLaunch = 8;
constexpr int kTieCap = 1024;

// Per-tile record, built on the host: the tile's samples [i0, e), its shard,
// the shard's first tile and first microbatch slot.
struct TileInfo {
  int64_t i0, e, mb_base;
  int32_t t_first, shard;
};

struct RoundsArgs {
  // the call's input: the stage [tables | sample_id | prompt_len | accepted],
  // copied to the device by one DMA before the first launch
  const uint64_t* in_id;
  const int32_t* in_prompt;
  const uint8_t* in_acc;
  const uint64_t* tables;    // [shard_off | mb_off | tiles] words (device)
  const uint64_t* tables_src;  // non-null: phase 1 reads the tables here (mapped host)
  int64_t table_words;         //   and CTA 0 copies them into `tables` for phase 2
  bool from_stage;           // first launch: build the state from the stage; else `snap`
  // device state
  yatt_sample* snap;         // state at the start of this launch (kept for re-runs)
  yatt_sample* work;         // final state of this launch
  int32_t* fate;             // [n] see kFate*
  int32_t* first_dev;        // [n] out_len after the launch's first round
  int64_t n, ntiles, slots;
  int32_t nshards, first_rank;
  uint64_t step;
  int32_t first_round, round_limit;
  yatt_round_params prm;
  double band;
  // device scratch
  int32_t* tile_cnt;          // [round_limit][ntiles]: pending per tile at each round's start
  yatt_round_report* rep;     // [round_limit][nshards]
  yatt_mb_agg* mbs;           // [round_limit][slots]
  unsigned* bar;              // [0] grid barrier (monotone, base below), [1] uncertified
                              // draws, [2] rounds this launch runs (both reset at the end)
  unsigned bar_base;
  uint64_t* tie_key;          // [kTieCap]
  const uint64_t* ovr_key;    // sorted
  const int32_t* ovr_len;
  int32_t n_ovr;
  // host (mapped) outputs, written once at the end
  int32_t* o_len;
  int32_t* o_round;
  uint8_t* o_acc;
  int32_t* o_first;           // nullable
  yatt_round_report* rep_out;  // [rounds_run][nshards] (num_microbatches: set by the host)
  yatt_mb_agg* mbs_out;        // [rounds_run][slots] raw slots (compacted by the host)
  uint64_t* tie_out;           // [kTieCap]
  int64_t* status;             // rounds_run, uncertified draws
  uint64_t* trace;             // nullable (device): %globaltimer of CTA 0 at phase boundaries
  uint64_t* trace_out;
};

// fate[i]: the round (index within the launch) in which sample i is
// accepted, | kFateForced when the acceptance was forced by max_rounds;
// round_limit if it is still pending after the launch; kFateDone if it was
// accepted before.  Acceptance never depends on the drawn lengths (the keyed
// rejection test of simcore.cpp:187-198 uses only ids and the round), so
// every sample's whole trajectory is known before any length is drawn.
constexpr int32_t kFateDone = -1;
constexpr int32_t kFateForced = 1 << 30;
constexpr int32_t kFateMask = kFateForced - 1;

__device__ __forceinline__ const int64_t* mb_off(const RoundsArgs& a) {
  return reinterpret_cast<const int64_t*>(a.tables) + a.nshards + 1;
}
__device__ __forceinline__ const TileInfo* tiles(const uint64_t* t, int32_t nshards) {
  return reinterpret_cast<const TileInfo*>(t + ((2 * nshards + 1 + 3) & ~3));
}

__device__ __forceinline__ void trace_mark(const RoundsArgs& a, int k) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && k < 30) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[k] = t;
  }
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier over a cooperative launch: a monotone arrival counter
// (the host tracks its base across launches, so nothing is reset per call).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {  // bar.sync orders the CTA's writes before this release
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (int(ld_acquire_u32(bar) - target) < 0) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ yatt_sample load_cg(const yatt_sample* p) {
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(p);
  unsigned long long v[3] = {__ldcg(w), __ldcg(w + 1), __ldcg(w + 2)};
  yatt_sample s;
  memcpy(&s, v, sizeof(s));
  return s;
}

__device__ __forceinline__ TileInfo load_tile(const TileInfo* p) {
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(p);
  unsigned long long v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = __ldg(w + q);
  TileInfo t;
  memcpy(&t, v, sizeof(t));
  return t;
}

__device__ __forceinline__ int draw_length(const RoundsArgs& a, int32_t round, int64_t idx,
                                           uint64_t id) {
  bool tie = false;
  const int len = length_keyed_dev(a.prm.out_dist, a.prm.seed, kOutputLenStream, a.step,
                                   uint64_t(int64_t(round)), id, a.band, &tie);
  if (!tie) return len;
  const uint64_t key = (uint64_t(uint32_t(round)) << 40) | uint64_t(idx);
  int lo = 0, hi = a.n_ovr - 1;
  while (lo <= hi) {  // host (glibc) value from an earlier pass of this call
    const int mid = (lo + hi) >> 1;
    const uint64_t k = a.ovr_key[mid];
    if (k == key) return a.ovr_len[mid];
    if (k < key) lo = mid + 1; else hi = mid - 1;
  }
  const unsigned slot = atomicAdd(a.bar + 1, 1u);
  if (slot < unsigned(kTieCap)) a.tie_key[slot] = key;
  return len;  // provisional: the host re-runs the call with the glibc value
}

__global__ void __launch_bounds__(kTile) rollout_rounds_kernel(const RoundsArgs a) {
  constexpr int kW = kTile / 32;
  __shared__ int s_wcnt[kW];
  __shared__ int s_wpart[kW][kRoundsPerLaunch];
  __shared__ int s_base[kRoundsPerLaunch];
  __shared__ long long s_part[kW][5];  // per warp: accepted, forced, pending, score, units
  __shared__ int s_len[kTile];         // by in-tile pending rank
  __shared__ long long s_tok[kTile];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int32_t mb = a.prm.microbatch_size;
  const int64_t gstride = int64_t(gridDim.x) * kTile;
  const int K = a.round_limit;  // <= kRoundsPerLaunch
  unsigned target = a.bar_base;
  int mark = 0;
  trace_mark(a, mark++);

  // ---- phase 1: every pending sample's fate (keyed rejection per round),
  // the pending count of every tile at the start of every round, the rounds
  // this launch needs; all rounds' report / microbatch slots initialised.
  const uint64_t* tab1 = a.tables_src ? a.tables_src : a.tables;
  if (a.tables_src && blockIdx.x == 0)  // zero-copy input: the device copy of the tables
    for (int64_t k = tid; k < a.table_words; k += kTile)
      const_cast<uint64_t*>(a.tables)[k] = a.tables_src[k];
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const TileInfo ti = load_tile(tiles(tab1, a.nshards) + t);
    const int64_t i = ti.i0 + tid;
    yatt_sample x{};
    if (i < ti.e)
      x = a.from_stage ? yatt_sample{a.in_id[i], a.in_prompt[i], 0, 0, int32_t(a.in_acc[i] != 0)}
                       : a.snap[i];
    int32_t fate = kFateDone;
    if (i < ti.e && x.accepted == 0) {
      const yatt_rejection_config& rc = a.prm.rejection;
      const uint64_t unit = rc.per_group ? x.sample_id / uint64_t(rc.group_size) : x.sample_id;
      fate = K;
      for (int ri = 0; ri < K; ++ri) {
        const int32_t round = a.first_round + ri;
        const bool rej = uniform_from_key(hash5(a.prm.seed, kRejectionStream, a.step,
                                                uint64_t(int64_t(round)), unit)) < rc.reject_rate;
        if (!rej || round >= a.prm.max_rounds) {
          fate = ri | (rej ? kFateForced : 0);
          break;
        }
      }
    }
    if (i < ti.e) {
      if (a.from_stage) a.snap[i] = x;
      a.work[i] = x;
      a.fate[i] = fate;
    }
    const int need = fate == kFateDone ? 0 : min((fate & kFateMask) + 1, K);
    int nmax = need;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    if (lane == 0 && nmax > 0) atomicMax(a.bar + 2, unsigned(nmax));
    for (int ri = 0; ri < K; ++ri) {
      const int c = __syncthreads_count(fate != kFateDone && (fate & kFateMask) >= ri);
      if (tid == 0) a.tile_cnt[int64_t(ri) * a.ntiles + t] = c;
    }
  }
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < int64_t(K) * a.nshards; j += gstride) {
    const int64_t ri = j / a.nshards, s = j - ri * a.nshards;
    a.rep[j] = yatt_round_report{a.first_rank + int32_t(s), a.first_round + int32_t(ri),
                                 0, 0, 0, 0, 0, 0, 0};
  }
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < int64_t(K) * a.slots; j += gstride)
    a.mbs[j] = yatt_mb_agg{0, 0, 0, 0, 0};
  trace_mark(a, mark++);
  grid_barrier(a.bar, target);
  trace_mark(a, mark++);

  // ---- phase 2: every round of every tile, no barrier between rounds.
  const int R = max(1, int(__ldcg(a.bar + 2)));  // rounds this launch runs
  const TileInfo* tile_tab = tiles(a.tables, a.nshards);
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const TileInfo ti = load_tile(tile_tab + t);
    const int s = ti.shard;
    const int64_t i = ti.i0 + tid;
    // pending samples of this shard in earlier tiles, at each round's start
    int c[kRoundsPerLaunch];
#pragma unroll
    for (int ri = 0; ri < kRoundsPerLaunch; ++ri) c[ri] = 0;
    for (int64_t k = ti.t_first + tid; k < t; k += kTile)
#pragma unroll
      for (int ri = 0; ri < kRoundsPerLaunch; ++ri)
        if (ri < R) c[ri] += __ldcg(a.tile_cnt + int64_t(ri) * a.ntiles + k);
#pragma unroll
    for (int ri = 0; ri < kRoundsPerLaunch; ++ri) {
      const int v = warp_sum(c[ri]);
      if (lane == 0) s_wpart[w][ri] = v;
    }
    yatt_sample x{};
    int32_t fate = kFateDone;
    if (i < ti.e) {
      x = load_cg(a.work + i);
      fate = __ldcg(a.fate + i);
    }
    __syncthreads();
    if (tid < R) {
      int b = 0;
#pragma unroll
      for (int k = 0; k < kW; ++k) b += s_wpart[k][tid];
      s_base[tid] = b;
    }
    const int acc_ri = fate & kFateMask;
    for (int ri = 0; ri < R; ++ri) {
      const int32_t round = a.first_round + ri;
      const bool pending = fate != kFateDone && acc_ri >= ri;
      const unsigned bal = __ballot_sync(0xffffffffu, pending);
      if (lane == 0) s_wcnt[w] = __popc(bal);
      __syncthreads();
      const int before_tile = s_base[ri];
      int rank = __popc(bal & ((1u << lane) - 1u)), n_pend = 0;
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        rank += k < w ? s_wcnt[k] : 0;
        n_pend += s_wcnt[k];
      }
      long long v[5] = {0, 0, 0, 0, 0};
      if (pending) {
        x.out_len_tokens = draw_length(a, round, i, x.sample_id);
        const long long tok = (long long)x.prompt_len_tokens + x.out_len_tokens;
        s_len[rank] = x.out_len_tokens;
        s_tok[rank] = tok;
        if (ri == 0) a.first_dev[i] = x.out_len_tokens;
        if (acc_ri == ri) {
          v[0] = 1;
          v[1] = (fate & kFateForced) ? 1 : 0;
          v[3] = tok;
          v[4] = tok * tok;
          x.accepted = 1;
          x.accepted_round = round;
        } else {
          v[2] = 1;
        }
      }
#pragma unroll
      for (int f = 0; f < 5; ++f) v[f] = warp_sum(v[f]);
      if (lane == 0) {
#pragma unroll
        for (int f = 0; f < 5; ++f) s_part[w][f] = v[f];
      }
      __syncthreads();
      // microbatch aggregates: the tile's pending run occupies positions
      // before_tile .. before_tile + n_pend of the shard's pending list; a
      // segmented suffix reduction per warp (segments = microbatches,
      // contiguous in rank order) leaves each segment's partial in its first
      // lane, which issues the three atomics (exact, order-free)
      if (w * 32 < n_pend) {
        const bool valid = tid < n_pend;
        const int seg = valid ? (before_tile + tid) / mb : INT_MAX;
        int cnt = valid ? 1 : 0, mx = valid ? s_len[tid] : 0;
        long long sc = valid ? s_tok[tid] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int oseg = __shfl_down_sync(0xffffffffu, seg, o);
          const int ocnt = __shfl_down_sync(0xffffffffu, cnt, o);
          const int omx = __shfl_down_sync(0xffffffffu, mx, o);
          const long long osc = __shfl_down_sync(0xffffffffu, sc, o);
          if (lane + o < 32 && oseg == seg) {
            cnt += ocnt;
            mx = max(mx, omx);
            sc += osc;
          }
        }
        const int pseg = __shfl_up_sync(0xffffffffu, seg, 1);
        if (valid && (lane == 0 || pseg != seg)) {
          yatt_mb_agg* m = a.mbs + int64_t(ri) * a.slots + ti.mb_base + seg;
          atomicAdd(&m->sample_count, cnt);
          atomicMax(&m->max_out_len_tokens, mx);
          atomicAdd(reinterpret_cast<unsigned long long*>(&m->score_tokens), (unsigned long long)sc);
        }
      }
      if (tid == 0 && n_pend) {
        long long tot[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < kW; ++k)
#pragma unroll
          for (int f = 0; f < 5; ++f) tot[f] += s_part[k][f];
        yatt_round_report* r = a.rep + int64_t(ri) * a.nshards + s;
        atomicAdd(&r->active_count, n_pend);
        atomicAdd(&r->newly_accepted_count, int(tot[0]));
        atomicAdd(&r->forced_accept_count, int(tot[1]));
        atomicAdd(&r->pending_count, int(tot[2]));
        atomicAdd(reinterpret_cast<unsigned long long*>(&r->accepted_score_tokens),
                  (unsigned long long)tot[3]);
        atomicAdd(reinterpret_cast<unsigned long long*>(&r->accepted_train_units),
                  (unsigned long long)tot[4]);
      }
      __syncthreads();  // shared arrays are reused by the next round / tile
    }
    if (fate != kFateDone) a.work[i] = x;
  }
  trace_mark(a, mark++);
  grid_barrier(a.bar, target);
  trace_mark(a, mark++);

  // ---- results into mapped host memory (zero-copy), once: stores to system
  // memory queue behind PCIe, so none are issued inside the rounds.
  for (int64_t i = int64_t(blockIdx.x) * kTile + tid; i < a.n; i += gstride) {
    const yatt_sample x = load_cg(a.work + i);
    a.o_len[i] = x.out_len_tokens;
    a.o_round[i] = x.accepted_round;
    a.o_acc[i] = uint8_t(x.accepted);
    if (a.o_first != nullptr) a.o_first[i] = __ldcg(a.first_dev + i);
  }
  const int64_t nrep = int64_t(R) * a.nshards;
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < nrep; j += gstride) {
    const long long* src = reinterpret_cast<const long long*>(a.rep + j);
    long long* dst = reinterpret_cast<long long*>(a.rep_out + j);
#pragma unroll
    for (int q = 0; q < int(sizeof(yatt_round_report) / 8); ++q) dst[q] = __ldcg(src + q);
  }
  const int64_t nslot = int64_t(R) * a.slots;
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < nslot; j += gstride) {
    const long long* src = reinterpret_cast<const long long*>(a.mbs + j);
    long long* dst = reinterpret_cast<long long*>(a.mbs_out + j);
    const long long cm = __ldcg(src + 1);  // sample_count | max_out_len
    if (cm != 0) {  // occupied slots only: the host reads the first nmb of each
      dst[1] = cm;
      dst[2] = __ldcg(src + 2);  // score_tokens (rank / index: the host)
    }
  }
  const unsigned ties = __ldcg(a.bar + 1);
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < min(int64_t(ties), int64_t(kTieCap));
       j += gstride)
    a.tie_out[j] = __ldcg(a.tie_key + j);
  trace_mark(a, mark++);
  if (blockIdx.x == 0 && tid == 0) {
    a.status[0] = R;
    a.status[1] = ties;
    a.bar[1] = 0;  // no CTA touches these counters after the last barrier
    a.bar[2] = 0;
  }
  if (a.trace && blockIdx.x == 0 && tid < 30) a.trace_out[tid] = a.trace[tid];
}

// Mapped pinned host buffer, grow-only.
struct HostBuf {
  void* h = nullptr;
  void* d = nullptr;
  size_t bytes = 0;
  int reserve(size_t need) {
    if (need <= bytes) return YATT_OK;
    if (h) cudaFreeHost(h);
    h = d = nullptr;
    bytes = 0;
    need = std::max<size_t>(need, 256);
    YATT_TRY_CUDA(cudaHostAlloc(&h, need, cudaHostAllocMapped));
    YATT_TRY_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    bytes = need;
    return YATT_OK;
  }
  ~HostBuf() {
    if (h) cudaFreeHost(h);
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int reserve(size_t need) {
    if (need <= bytes) return YATT_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    need = std::max<size_t>(need, 256);
    YATT_TRY_CUDA(cudaMalloc(&p, need));
    bytes = need;
    return YATT_OK;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Staging layout (mapped host): tables [shard_off (nshards+1) | mb_off (nshards)
// | pad to 32 B | TileInfo (<= n/256 + nshards)] then the SoA input and output
// arrays of n samples.
struct StageLayout {
  size_t tables, words, id, prompt, acc, o_len, o_round, o_acc, o_first, end;
  StageLayout(int64_t n, int32_t nshards) {
    const size_t head = size_t((2 * nshards + 1 + 3) & ~3) * 8;
    words = (head + sizeof(TileInfo) * size_t(n / kTile + nshards)) / 8;
    tables = 0;
    id = align_up(words * 8);
    prompt = id + align_up(8 * size_t(n));
    acc = prompt + align_up(4 * size_t(n));
    o_len = acc + align_up(size_t(n));
    o_round = o_len + align_up(4 * size_t(n));
    o_acc = o_round + align_up(4 * size_t(n));
    o_first = o_acc + align_up(size_t(n));
    end = o_first + align_up(4 * size_t(n));
  }
};

}  // namespace
}  // namespace yattb

using namespace yattb;

struct yatt_rounds {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  HostBuf stage;   // tables + SoA input/output of the call (mapped)
  HostBuf outs;    // reports / microbatches / status of one launch (mapped)
  DevBuf dev;      // device state + scratch
  DevBuf ovr_dev;  // glibc overrides of uncertified draws (separate: may grow between re-runs)
  unsigned bar_base = 0;  // arrivals so far on the grid-barrier counter
  bool bar_valid = false;
  int grid_cap = 0;
  int64_t staged_n = -1;
  int32_t staged_shards = 0;
  DevBuf xin, xout;  // yatt_peer_rounds_run: the exchange's device words
  // accumulated over the launches of one call
  std::vector<yatt_round_report> reps;
  std::vector<yatt_mb_agg> mbs;
  int64_t n = 0, redrawn = 0;
  int32_t rounds = 0, nshards = 0;
  bool have_first = false;
};

extern "C" {

int yatt_rounds_create(yatt_rounds_t* out) {
  YATT_REQUIRE(out != nullptr, YATT_ERR_CONFIG, "rounds_create: null handle pointer");
  auto* h = new yatt_rounds();
  cudaGetDevice(&h->device);
  const cudaError_t e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete h;
    return set_error(YATT_ERR_CUDA, "rounds_create: %s", cudaGetErrorString(e));
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rollout_rounds_kernel, kTile, 0);
  h->grid_cap = std::max(1, per_sm) * num_sms();
  *out = h;
  return YATT_OK;
}

void yatt_rounds_destroy(yatt_rounds_t h) {
  if (!h) return;
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
}

int yatt_rounds_stage(yatt_rounds_t h, int64_t n, int32_t nshards, yatt_rounds_io* io) {
  YATT_REQUIRE(h != nullptr && io != nullptr, YATT_ERR_CONFIG, "rounds_stage: null argument");
  YATT_REQUIRE(n >= 0 && nshards >= 1, YATT_ERR_CONFIG, "rounds_stage: bad sizes");
  const StageLayout L(n, nshards);
  int rc = h->stage.reserve(L.end);
  if (rc) return rc;
  char* b = static_cast<char*>(h->stage.h);
  io->sample_id = reinterpret_cast<uint64_t*>(b + L.id);
  io->prompt_len = reinterpret_cast<int32_t*>(b + L.prompt);
  io->accepted = reinterpret_cast<uint8_t*>(b + L.acc);
  io->out_len = reinterpret_cast<int32_t*>(b + L.o_len);
  io->accepted_round = reinterpret_cast<int32_t*>(b + L.o_round);
  io->accepted_out = reinterpret_cast<uint8_t*>(b + L.o_acc);
  io->first_round_len = reinterpret_cast<int32_t*>(b + L.o_first);
  h->staged_n = n;
  h->staged_shards = nshards;
  return YATT_OK;
}

int yatt_rounds_run(yatt_rounds_t h, int64_t n, const int64_t* h_shard_offsets, int32_t nshards,
                    int32_t first_rank, int32_t step_index, int32_t first_round,
                    int32_t round_limit, const yatt_round_params* prm, int32_t want_first_lens,
                    void* stream) {
  YATT_REQUIRE(h != nullptr && prm != nullptr && h_shard_offsets != nullptr, YATT_ERR_CONFIG,
               "rounds_run: null argument");
  YATT_REQUIRE(prm->microbatch_size > 0, YATT_ERR_CONFIG, "microbatch_size must be positive");
  YATT_REQUIRE(prm->out_dist.kind >= 0 && prm->out_dist.kind <= 3, YATT_ERR_CONFIG,
               "unknown distribution kind value");
  YATT_REQUIRE(!prm->rejection.per_group || prm->rejection.group_size > 0, YATT_ERR_CONFIG,
               "group_size must be positive for per-group rejection");
  YATT_REQUIRE(nshards >= 1 && n >= 0, YATT_ERR_CONFIG, "rounds_run: bad sizes");
  YATT_REQUIRE(h->staged_n == n && h->staged_shards == nshards, YATT_ERR_CONFIG,
               "rounds_run: stage %lld samples / %d shards with yatt_rounds_stage first",
               (long long)n, nshards);
  YATT_REQUIRE(h_shard_offsets[0] == 0 && h_shard_offsets[nshards] == n, YATT_ERR_CONFIG,
               "rounds_run: shard offsets must span [0, n)");
  YATT_REQUIRE(n < (int64_t(1) << 40), YATT_ERR_CONFIG, "rounds_run: too many samples");
  int dev_now = 0;
  YATT_TRY_CUDA(cudaGetDevice(&dev_now));
  YATT_REQUIRE(dev_now == h->device, YATT_ERR_CONFIG, "rounds_run: handle belongs to device %d",
               h->device);
  cudaStream_t st = stream ? as_stream(stream) : h->own_stream;
  const StageLayout L(n, nshards);
  char* sb = static_cast<char*>(h->stage.h);
  char* sd = static_cast<char*>(h->stage.d);

  // shard / tile tables into the staging head
  int64_t* t_shard = reinterpret_cast<int64_t*>(sb);
  int64_t* t_mb = t_shard + nshards + 1;
  TileInfo* t_tiles = reinterpret_cast<TileInfo*>(sb + size_t((2 * nshards + 1 + 3) & ~3) * 8);
  int64_t ntiles = 0, slots = 0;
  for (int32_t s = 0; s < nshards; ++s) {
    const int64_t b = h_shard_offsets[s], sz = h_shard_offsets[s + 1] - b;
    YATT_REQUIRE(sz >= 0, YATT_ERR_CONFIG, "shard offsets must ascend");
    YATT_REQUIRE(sz < (int64_t(1) << 31), YATT_ERR_CONFIG, "rounds_run: shard too large");
    t_shard[s] = b;
    t_mb[s] = slots;
    const int64_t t_first = ntiles;
    for (int64_t k = 0; k < ceil_div(sz, kTile); ++k)
      t_tiles[ntiles++] = TileInfo{b + k * kTile, b + sz, slots, int32_t(t_first), s};
    slots += ceil_div(sz, prm->microbatch_size);
  }
  t_shard[nshards] = n;

  const int32_t limit = round_limit > 0 ? round_limit : INT32_MAX;
  const int32_t K = std::min(kRoundsPerLaunch, limit);
  const size_t ss = sizeof(yatt_sample) * size_t(n);
  // device: [stage input copy | snap | work | first | tile_cnt | rep | mbs | pair_base | ties | trace]
  const size_t in_bytes = L.o_len;  // tables + sample_id + prompt_len + accepted
  const size_t o_snap = align_up(in_bytes);
  const size_t o_work = o_snap + align_up(ss);
  const size_t o_first = o_work + align_up(ss);
  const size_t o_fate = o_first + align_up(4 * size_t(n));
  const size_t o_tile = o_fate + align_up(4 * size_t(n));
  const size_t o_rep = o_tile + align_up(sizeof(int32_t) * size_t(K) * size_t(ntiles));
  const size_t o_mbs = o_rep + align_up(sizeof(yatt_round_report) * size_t(K) * nshards);
  const size_t o_ties = o_mbs + align_up(sizeof(yatt_mb_agg) * size_t(K) * size_t(slots));
  const size_t o_trace = o_ties + align_up(sizeof(uint64_t) * kTieCap);
  const size_t o_end = o_trace + 256;
  // outputs (mapped): [reps | mbs | ties | status | trace]
  const size_t p_mbs = align_up(sizeof(yatt_round_report) * size_t(K) * nshards);
  const size_t p_ties = p_mbs + align_up(sizeof(yatt_mb_agg) * size_t(K) * size_t(slots));
  const size_t p_status = p_ties + align_up(sizeof(uint64_t) * kTieCap);
  const size_t p_end = p_status + 64 + 32 * 8;
  int rc = h->outs.reserve(p_end);
  if (rc) return rc;
  if (o_end > h->dev.bytes) h->bar_valid = false;  // fresh scratch: counters are garbage
  rc = h->dev.reserve(o_end);
  if (rc) return rc;
  // the barrier / draw counters live in a small fixed block at the end of the
  // stage-independent region: put them in the ovr buffer's head instead
  rc = h->ovr_dev.reserve(256);
  if (rc) return rc;
  if (!h->bar_valid) {
    YATT_TRY_CUDA(cudaMemsetAsync(h->ovr_dev.p, 0, 8, st));
    h->bar_base = 0;
    h->bar_valid = true;
  }

  h->reps.clear();
  h->mbs.clear();
  h->n = n;
  h->nshards = nshards;
  h->rounds = 0;
  h->redrawn = 0;
  h->have_first = false;
  const uint64_t* h_id = reinterpret_cast<const uint64_t*>(sb + L.id);
  std::map<uint64_t, int32_t> ovr;  // (round << 40 | index) -> glibc length
  int32_t round = first_round;
  bool first_launch = true, staged = false;
  char* ob = static_cast<char*>(h->outs.h);
  char* od = static_cast<char*>(h->outs.d);
  char* db = static_cast<char*>(h->dev.p);
  static const bool tracing = std::getenv("YATT_ROUNDS_TRACE") != nullptr;
  static const bool zero_copy = [] {
    const char* e = std::getenv("YATT_ROUNDS_ZC");
    return e == nullptr || std::atoi(e) != 0;
  }();


  while (true) {
    const size_t ovr_bytes = 256 + align_up(8 * ovr.size()) + align_up(4 * ovr.size());
    if (ovr_bytes > h->ovr_dev.bytes) {  // grow, keeping the counters
      unsigned keep[2];
      YATT_TRY_CUDA(cudaMemcpyAsync(keep, h->ovr_dev.p, 8, cudaMemcpyDeviceToHost, st));
      YATT_TRY_CUDA(cudaStreamSynchronize(st));
      rc = h->ovr_dev.reserve(ovr_bytes);
      if (rc) return rc;
      YATT_TRY_CUDA(cudaMemcpyAsync(h->ovr_dev.p, keep, 8, cudaMemcpyHostToDevice, st));
    }
    char* dov = static_cast<char*>(h->ovr_dev.p);
    if (!ovr.empty()) {
      std::vector<uint64_t> k;
      std::vector<int32_t> v;
      for (const auto& kv : ovr) {
        k.push_back(kv.first);
        v.push_back(kv.second);
      }
      YATT_TRY_CUDA(cudaMemcpyAsync(dov + 256, k.data(), 8 * k.size(), cudaMemcpyHostToDevice, st));
      YATT_TRY_CUDA(cudaMemcpyAsync(dov + 256 + align_up(8 * k.size()), v.data(), 4 * v.size(),
                                    cudaMemcpyHostToDevice, st));
      YATT_TRY_CUDA(cudaStreamSynchronize(st));  // k, v are stack-owned
    }
    const auto th0 = std::chrono::steady_clock::now();
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    if (tracing) {
      for (auto& e : ev) cudaEventCreate(&e);
      cudaEventRecord(ev[0], st);
    }
    // the packed input: read in place from the mapped stage by the first
    // launch (zero-copy: no DMA to set up; round loop 0.092 vs 0.096 ms at
    // configs[4]), or one DMA (YATT_ROUNDS_ZC=0)
    if (!zero_copy && first_launch && !staged) {
      YATT_TRY_CUDA(cudaMemcpyAsync(db, sb, in_bytes, cudaMemcpyHostToDevice, st));
      staged = true;
    }
    if (tracing) cudaEventRecord(ev[1], st);
    RoundsArgs a{};
    const char* ib = zero_copy ? sd : db;
    a.in_id = reinterpret_cast<const uint64_t*>(ib + L.id);
    a.in_prompt = reinterpret_cast<const int32_t*>(ib + L.prompt);
    a.in_acc = reinterpret_cast<const uint8_t*>(ib + L.acc);
    a.tables = reinterpret_cast<const uint64_t*>(db);
    a.tables_src = zero_copy && first_launch ? reinterpret_cast<const uint64_t*>(sd) : nullptr;
    a.table_words = int64_t(L.words);
    a.from_stage = first_launch;
    a.snap = reinterpret_cast<yatt_sample*>(db + o_snap);
    a.work = reinterpret_cast<yatt_sample*>(db + o_work);
    a.first_dev = reinterpret_cast<int32_t*>(db + o_first);
    a.fate = reinterpret_cast<int32_t*>(db + o_fate);
    a.n = n;
    a.ntiles = ntiles;
    a.slots = slots;
    a.nshards = nshards;
    a.first_rank = first_rank;
    a.step = uint64_t(int64_t(step_index));
    a.first_round = round;
    a.round_limit = int32_t(std::min<int64_t>(K, int64_t(limit) - (round - first_round)));
    a.prm = *prm;
    a.band = g_tie_band;
    a.tile_cnt = reinterpret_cast<int32_t*>(db + o_tile);
    a.rep = reinterpret_cast<yatt_round_report*>(db + o_rep);
    a.mbs = reinterpret_cast<yatt_mb_agg*>(db + o_mbs);
    a.bar = reinterpret_cast<unsigned*>(dov);
    a.bar_base = h->bar_base;
    a.tie_key = reinterpret_cast<uint64_t*>(db + o_ties);
    a.ovr_key = reinterpret_cast<const uint64_t*>(dov + 256);
    a.ovr_len = reinterpret_cast<const int32_t*>(dov + 256 + align_up(8 * ovr.size()));
    a.n_ovr = int32_t(ovr.size());
    a.o_len = reinterpret_cast<int32_t*>(sd + L.o_len);
    a.o_round = reinterpret_cast<int32_t*>(sd + L.o_round);
    a.o_acc = reinterpret_cast<uint8_t*>(sd + L.o_acc);
    a.o_first = (want_first_lens && first_launch) ? reinterpret_cast<int32_t*>(sd + L.o_first) : nullptr;
    a.rep_out = reinterpret_cast<yatt_round_report*>(od);
    a.mbs_out = reinterpret_cast<yatt_mb_agg*>(od + p_mbs);
    a.tie_out = reinterpret_cast<uint64_t*>(od + p_ties);
    a.status = reinterpret_cast<int64_t*>(od + p_status);
    a.trace = tracing ? reinterpret_cast<uint64_t*>(db + o_trace) : nullptr;
    a.trace_out = reinterpret_cast<uint64_t*>(od + p_status + 64);
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ntiles, h->grid_cap)));
    void* args[] = {&a};
    h->bar_valid = false;  // until the launch is known to have completed
    YATT_TRY_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(rollout_rounds_kernel),
                                              dim3(grid), dim3(kTile), args, 0, st));
    if (tracing) cudaEventRecord(ev[2], st);
    const auto th1 = std::chrono::steady_clock::now();
    YATT_TRY_CUDA(cudaStreamSynchronize(st));
    const auto th2 = std::chrono::steady_clock::now();
    const int64_t* status = reinterpret_cast<const int64_t*>(ob + p_status);
    const int32_t rr = int32_t(status[0]);
    h->bar_base += unsigned(grid) * 2u;  // two grid barriers per launch
    h->bar_valid = true;
    if (a.trace) {
      const uint64_t* tr = reinterpret_cast<const uint64_t*>(ob + p_status + 64);
      using us = std::chrono::duration<double, std::micro>;
      float e01 = 0, e12 = 0;
      cudaEventElapsedTime(&e01, ev[0], ev[1]);
      cudaEventElapsedTime(&e12, ev[1], ev[2]);
      for (auto& e : ev) cudaEventDestroy(e);
      std::fprintf(stderr, "[host us] copy+launch %.1f sync %.1f [events us] dma %.1f kernel %.1f | ",
                   us(th1 - th0).count(), us(th2 - th1).count(), e01 * 1e3, e12 * 1e3);
      std::fprintf(stderr, "[rounds trace us]");
      for (int k = 1; k < 30; ++k)
        if (tr[k] > tr[0]) std::fprintf(stderr, " %d:%.2f", k, (tr[k] - tr[0]) * 1e-3);
      std::fprintf(stderr, "\n");
      std::memset(const_cast<uint64_t*>(tr), 0, 32 * 8);
    }
    const int64_t ties = status[1];
    if (ties > 0) {  // redo the uncertified draws with glibc and re-run this launch
      const uint64_t* keys = reinterpret_cast<const uint64_t*>(ob + p_ties);
      for (int64_t j = 0; j < std::min<int64_t>(ties, kTieCap); ++j) {
        const uint64_t key = keys[j];
        const int64_t idx = int64_t(key & ((uint64_t(1) << 40) - 1));
        ovr[key] = length_keyed_glibc(prm->out_dist, prm->seed, kOutputLenStream,
                                      uint64_t(int64_t(step_index)), key >> 40, h_id[idx]);
      }
      h->redrawn = int64_t(ovr.size());
      continue;  // the kernel never writes `snap`: the re-run starts from the same state
    }
    // reports in round-major order; microbatches compacted from the raw
    // slots: ceil(active / microbatch_size) per report, rank + index filled in
    const auto* rp = reinterpret_cast<const yatt_round_report*>(ob);
    const auto* mp = reinterpret_cast<const yatt_mb_agg*>(ob + p_mbs);
    for (int32_t r = 0; r < rr; ++r)
      for (int32_t s = 0; s < nshards; ++s) {
        yatt_round_report rep = rp[int64_t(r) * nshards + s];
        rep.num_microbatches = ceil_div(rep.active_count, prm->microbatch_size);
        const yatt_mb_agg* raw = mp + int64_t(r) * slots + t_mb[s];
        for (int64_t q = 0; q < rep.num_microbatches; ++q)
          h->mbs.push_back(yatt_mb_agg{first_rank + s, int32_t(q), raw[q].sample_count,
                                       raw[q].max_out_len_tokens, raw[q].score_tokens});
        h->reps.push_back(rep);
      }
    if (a.o_first) h->have_first = true;
    h->rounds += rr;
    round += rr;
    bool more = false;
    for (int32_t s = 0; s < nshards; ++s) more |= rp[int64_t(rr - 1) * nshards + s].pending_count > 0;
    if (!more || round - first_round >= limit) break;
    // continue from this launch's final state
    YATT_TRY_CUDA(cudaMemcpyAsync(db + o_snap, db + o_work, ss, cudaMemcpyDeviceToDevice, st));
    first_launch = false;
  }
  return YATT_OK;
}

int yatt_rounds_result(yatt_rounds_t h, yatt_rounds_view* v) {
  YATT_REQUIRE(h != nullptr && v != nullptr, YATT_ERR_CONFIG, "rounds_result: null argument");
  v->reports = h->reps.data();
  v->rounds = h->rounds;
  v->num_shards = h->nshards;
  v->microbatches = h->mbs.data();
  v->num_microbatches = int64_t(h->mbs.size());
  v->redrawn_on_host = h->redrawn;
  v->first_round_lens_valid = h->have_first ? 1 : 0;
  return YATT_OK;
}

// The multi-rank step with ONE exchange (fates first: acceptance never
// depends on the drawn lengths, so every rank can run its own controller
// shard to completion without hearing from the others).  The global loop of
// the reference (simcore.cpp:470-490; the coordinator's continue test,
// demo.cpp:468-476) runs max-over-ranks rounds, a finished shard reporting
// zeros; this rank's reports + microbatch aggregates travel once, as int64
// words through the peer all-gather kernel, and the handle's result view
// becomes the GLOBAL one: reports[round][rank], microbatches in that order.
int yatt_peer_rounds_run(yatt_peer_t peer, yatt_rounds_t h, int64_t n, int32_t step_index,
                         const yatt_round_params* prm, int32_t want_first_lens, void* stream) {
  YATT_REQUIRE(h != nullptr && prm != nullptr, YATT_ERR_CONFIG, "peer_rounds_run: null argument");
  int32_t world = 0, rank = 0;
  int rc = yatt_peer_world(peer, &world, &rank);
  if (rc) return rc;
  const int64_t off[2] = {0, n};
  rc = yatt_rounds_run(h, n, off, 1, rank, step_index, 1, 0, prm, want_first_lens, stream);
  if (rc) return rc;
  // wire: [rounds, reports (6 words each), microbatches (3 words each)]
  static_assert(sizeof(yatt_round_report) == 48 && sizeof(yatt_mb_agg) == 24, "wire words");
  const int64_t R = h->rounds, M = int64_t(h->mbs.size());
  std::vector<int64_t> mine(size_t(1 + 6 * R + 3 * M));
  mine[0] = R;
  std::memcpy(mine.data() + 1, h->reps.data(), size_t(48 * R));
  std::memcpy(mine.data() + 1 + 6 * R, h->mbs.data(), size_t(24 * M));
  const cudaStream_t st = stream ? as_stream(stream) : h->own_stream;
  const int64_t cap = YATT_PEER_GATHER_MAX_WORDS;
  rc = h->xin.reserve(size_t(8 * cap));
  if (!rc) rc = h->xout.reserve(size_t(8 * cap * world));
  if (rc) return rc;
  int64_t* din = static_cast<int64_t*>(h->xin.p);
  int64_t* dout = static_cast<int64_t*>(h->xout.p);
  const int64_t my_words = int64_t(mine.size());
  std::vector<int64_t> sizes(static_cast<size_t>(world));
  YATT_TRY_CUDA(cudaMemcpyAsync(din, &my_words, 8, cudaMemcpyHostToDevice, st));
  rc = yatt_peer_allgather_i64(peer, din, 1, dout, st);
  if (rc) return rc;
  YATT_TRY_CUDA(cudaMemcpyAsync(sizes.data(), dout, 8 * size_t(world), cudaMemcpyDeviceToHost, st));
  YATT_TRY_CUDA(cudaStreamSynchronize(st));
  for (int32_t r = 0; r < world; ++r)  // a timed-out gather leaves -1 words (yatt_peer_status)
    YATT_REQUIRE(sizes[size_t(r)] >= 1 && sizes[size_t(r)] <= (int64_t(1) << 40), YATT_ERR_CUDA,
                 "peer_rounds_run: rank %d sent no report words (peer timeout?)", r);
  const int64_t width = *std::max_element(sizes.begin(), sizes.end());
  mine.resize(size_t(width), 0);
  std::vector<int64_t> all(size_t(world * width)), chunk(size_t(world * cap));
  for (int64_t c0 = 0; c0 < width; c0 += cap) {
    const int64_t cw = std::min(cap, width - c0);
    YATT_TRY_CUDA(cudaMemcpyAsync(din, mine.data() + c0, size_t(8 * cw), cudaMemcpyHostToDevice, st));
    rc = yatt_peer_allgather_i64(peer, din, int32_t(cw), dout, st);
    if (rc) return rc;
    YATT_TRY_CUDA(cudaMemcpyAsync(chunk.data(), dout, size_t(8 * cw * world), cudaMemcpyDeviceToHost,
                                  st));
    YATT_TRY_CUDA(cudaStreamSynchronize(st));
    for (int32_t r = 0; r < world; ++r)
      std::memcpy(all.data() + size_t(r * width + c0), chunk.data() + size_t(r * cw), size_t(8 * cw));
  }
  int32_t peer_status = 0;
  rc = yatt_peer_status(peer, &peer_status);
  if (rc) return rc;
  YATT_REQUIRE(peer_status == 0, YATT_ERR_CUDA,
               "peer_rounds_run: a rank did not arrive (peer all-gather timed out)");
  // the global view, round-major then rank
  int64_t rounds_g = 0;
  std::vector<int64_t> mb_cursor(static_cast<size_t>(world));
  for (int32_t r = 0; r < world; ++r) {
    const int64_t* w = all.data() + size_t(r * width);
    YATT_REQUIRE(w[0] >= 0 && 1 + 6 * w[0] <= sizes[size_t(r)], YATT_ERR_CUDA,
                 "peer_rounds_run: malformed words from rank %d", r);
    rounds_g = std::max(rounds_g, w[0]);
    mb_cursor[size_t(r)] = 1 + 6 * w[0];
  }
  h->reps.clear();
  h->mbs.clear();
  for (int64_t k = 0; k < rounds_g; ++k)
    for (int32_t r = 0; r < world; ++r) {
      const int64_t* w = all.data() + size_t(r * width);
      if (k < w[0]) {
        yatt_round_report rep;
        std::memcpy(&rep, w + 1 + 6 * k, 48);
        YATT_REQUIRE(rep.num_microbatches >= 0 &&
                         mb_cursor[size_t(r)] + 3 * rep.num_microbatches <= sizes[size_t(r)],
                     YATT_ERR_CUDA, "peer_rounds_run: malformed microbatches from rank %d", r);
        for (int64_t q = 0; q < rep.num_microbatches; ++q) {
          yatt_mb_agg m;
          std::memcpy(&m, w + mb_cursor[size_t(r)] + 3 * q, 24);
          h->mbs.push_back(m);
        }
        mb_cursor[size_t(r)] += 3 * rep.num_microbatches;
        h->reps.push_back(rep);
      } else {  // this shard finished earlier: the coordinator's zero report
        yatt_round_report z{};
        z.controller_rank = r;
        z.round = int32_t(k + 1);
        h->reps.push_back(z);
      }
    }
  h->rounds = int32_t(rounds_g);
  h->nshards = world;
  return YATT_OK;
}

int yatt_set_tie_band(double band) {
  YATT_REQUIRE(band >= 0 && band < 0.5, YATT_ERR_CONFIG, "tie band must lie in [0, 0.5)");
  g_tie_band = band;
  return YATT_OK;
}

}  // extern "C"
