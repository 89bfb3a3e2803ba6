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
// Kernel: a cooperative grid (every CTA resident), one 256-sample tile per
// CTA iteration.  Per round, two grid barriers:
//   phase 1  zero the round's report / microbatch slots; per tile, count the
//            samples still pending at round start
//   phase 2  per tile: base = pending count of the shard's earlier tiles,
//            in-tile order by ballot; draw, reject, update the sample,
//            integer atomics into the round's report and microbatch slots
//   phase 3  every CTA sums the shards' pending counts (same value in all
//            CTAs: the loop exits uniformly); CTA 0 sets num_microbatches and
//            the compacted output position of each (round, shard)
// After the last round: final sample state, the reports of the rounds run and
// the compacted microbatches are stored straight into mapped pinned host
// memory (zero-copy), so a call is: one H2D copy of the packed samples, one
// launch, one stream synchronize.
//
// Normal / LogNormal draws that are not certified equal to glibc
// (keyed_draw.cuh) are logged; the host recomputes exactly those with glibc
// and re-runs the call with them as overrides, so results are bit-exact with
// the reference by construction.
#include <cuda_runtime.h>

#include <algorithm>
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

struct RoundsArgs {
  const yatt_sample* in;     // device: state at the start of this launch
  yatt_sample* work;         // device
  yatt_sample* out;          // mapped host: final state
  int32_t* first_lens;       // mapped host (nullable): out_len after the launch's first round
  const int64_t* shard_off;  // device [nshards + 1]
  const int64_t* tile_off;   // device [nshards + 1]
  const int64_t* mb_off;     // device [nshards]
  int64_t n, ntiles, slots;
  int32_t nshards, first_rank;
  uint64_t step;
  int32_t first_round, round_limit;
  yatt_round_params prm;
  double band;
  // device scratch
  int32_t* tile_cnt;          // [ntiles]
  yatt_round_report* rep;     // [round_limit][nshards]
  yatt_mb_agg* mbs;           // [round_limit][slots]
  int64_t* pair_base;         // [round_limit][nshards]
  unsigned* bar;              // [0] grid barrier, [1] tie count (zeroed per launch)
  uint64_t* tie_key;          // [kTieCap]
  const uint64_t* ovr_key;    // sorted
  const int32_t* ovr_len;
  int32_t n_ovr;
  // mapped host outputs
  yatt_round_report* rep_out;  // [rounds_run][nshards]
  yatt_mb_agg* mbs_out;        // compacted, (round, shard, mb_index) order
  uint64_t* tie_out;           // [kTieCap]
  int64_t* status;             // rounds_run, n_mbs, ties
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier over a cooperative launch (monotone counter, zeroed
// before the launch).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire_u32(bar) < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

// Largest s in [0, n) with off[s] <= x (off ascending, off[0] <= x).
__device__ __forceinline__ int last_le(const int64_t* off, int n, int64_t x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(off + mid) <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  T s = 0;
#pragma unroll
  for (int k = 0; k < kTile / 32; ++k) s += red[k];
  __syncthreads();
  return s;
}

__device__ __forceinline__ yatt_sample load_cg(const yatt_sample* p) {
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(p);
  unsigned long long v[3] = {__ldcg(w), __ldcg(w + 1), __ldcg(w + 2)};
  yatt_sample s;
  memcpy(&s, v, sizeof(s));
  return s;
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
  __shared__ int s_red[kTile / 32];
  __shared__ long long s_red64[kTile / 32];
  __shared__ int s_wcnt[kTile / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int32_t mb = a.prm.microbatch_size;
  const int64_t gstride = int64_t(gridDim.x) * kTile;
  unsigned target = 0;

  for (int64_t i = int64_t(blockIdx.x) * kTile + tid; i < a.n; i += gstride) a.work[i] = a.in[i];
  grid_barrier(a.bar, target);

  int rounds_run = 0;
  long long cursor = 0;  // CTA 0: compacted microbatch count so far
  for (int ri = 0; ri < a.round_limit; ++ri) {
    const int32_t round = a.first_round + ri;
    const bool final_round = round >= a.prm.max_rounds;
    yatt_round_report* rep = a.rep + int64_t(ri) * a.nshards;
    yatt_mb_agg* mbs = a.mbs + int64_t(ri) * a.slots;

    // ---- phase 1 -------------------------------------------------------
    for (int64_t s = int64_t(blockIdx.x) * kTile + tid; s < a.nshards; s += gstride)
      rep[s] = yatt_round_report{a.first_rank + int32_t(s), round, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t k = int64_t(blockIdx.x) * kTile + tid; k < a.slots; k += gstride) {
      const int s = last_le(a.mb_off, a.nshards, k);
      mbs[k] = yatt_mb_agg{a.first_rank + s, int32_t(k - __ldg(a.mb_off + s)), 0, 0, 0};
    }
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      const int s = last_le(a.tile_off, a.nshards, t);
      const int64_t e = __ldg(a.shard_off + s + 1);
      const int64_t i = __ldg(a.shard_off + s) + (t - __ldg(a.tile_off + s)) * kTile + tid;
      const bool pend = i < e && __ldcg(&a.work[i].accepted) == 0;
      const int c = __syncthreads_count(pend);
      if (tid == 0) a.tile_cnt[t] = c;
    }
    grid_barrier(a.bar, target);

    // ---- phase 2 -------------------------------------------------------
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      const int s = last_le(a.tile_off, a.nshards, t);
      const int64_t t_first = __ldg(a.tile_off + s);
      const int64_t e = __ldg(a.shard_off + s + 1);
      const int64_t i = __ldg(a.shard_off + s) + (t - t_first) * kTile + tid;
      int c = 0;
      for (int64_t k = t_first + tid; k < t; k += kTile) c += __ldcg(a.tile_cnt + k);
      const int before_tile = block_sum(c, s_red);
      yatt_sample x{};
      bool pending = false;
      if (i < e) {
        x = load_cg(a.work + i);
        pending = x.accepted == 0;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, pending);
      if (lane == 0) s_wcnt[w] = __popc(bal);
      __syncthreads();
      int pos = before_tile + __popc(bal & ((1u << lane) - 1u));
      for (int k = 0; k < w; ++k) pos += s_wcnt[k];
      __syncthreads();
      int acc = 0, forced = 0, pend = 0;
      long long score = 0, units = 0;
      if (pending) {
        x.out_len_tokens = draw_length(a, round, i, x.sample_id);
        yatt_mb_agg* m = mbs + __ldg(a.mb_off + s) + pos / mb;
        atomicAdd(&m->sample_count, 1);
        atomicMax(&m->max_out_len_tokens, x.out_len_tokens);
        atomicAdd(reinterpret_cast<unsigned long long*>(&m->score_tokens),
                  (unsigned long long)(int64_t(x.prompt_len_tokens) + x.out_len_tokens));
        const yatt_rejection_config& rc = a.prm.rejection;
        const uint64_t unit = rc.per_group ? x.sample_id / uint64_t(rc.group_size) : x.sample_id;
        const bool rej = uniform_from_key(hash5(a.prm.seed, kRejectionStream, a.step,
                                                uint64_t(int64_t(round)), unit)) < rc.reject_rate;
        if (rej && !final_round) {
          pend = 1;
        } else {
          forced = rej ? 1 : 0;
          x.accepted = 1;
          x.accepted_round = round;
          acc = 1;
          const long long tok = (long long)x.prompt_len_tokens + x.out_len_tokens;
          score = tok;
          units = tok * tok;
        }
        a.work[i] = x;
      }
      if (ri == 0 && a.first_lens != nullptr && i < e) a.first_lens[i] = x.out_len_tokens;
      const int active = __syncthreads_count(pending);
      const int n_acc = block_sum(acc, s_red);
      const int n_forced = block_sum(forced, s_red);
      const int n_pend = block_sum(pend, s_red);
      const long long sc = block_sum(score, s_red64);
      const long long un = block_sum(units, s_red64);
      if (tid == 0 && active) {
        yatt_round_report* r = rep + s;
        atomicAdd(&r->active_count, active);
        atomicAdd(&r->newly_accepted_count, n_acc);
        atomicAdd(&r->forced_accept_count, n_forced);
        atomicAdd(&r->pending_count, n_pend);
        atomicAdd(reinterpret_cast<unsigned long long*>(&r->accepted_score_tokens),
                  (unsigned long long)sc);
        atomicAdd(reinterpret_cast<unsigned long long*>(&r->accepted_train_units),
                  (unsigned long long)un);
      }
    }
    grid_barrier(a.bar, target);

    // ---- phase 3 -------------------------------------------------------
    long long p = 0;
    for (int64_t s = tid; s < a.nshards; s += kTile) p += __ldcg(&rep[s].pending_count);
    const long long pending_total = block_sum(p, s_red64);
    if (blockIdx.x == 0 && tid == 0) {
      for (int32_t s = 0; s < a.nshards; ++s) {
        const int64_t nmb = (int64_t(__ldcg(&rep[s].active_count)) + mb - 1) / mb;
        rep[s].num_microbatches = nmb;
        a.pair_base[int64_t(ri) * a.nshards + s] = cursor;
        cursor += nmb;
      }
    }
    rounds_run = ri + 1;
    if (pending_total == 0) break;
  }
  grid_barrier(a.bar, target);

  // ---- copy-out into mapped host memory ---------------------------------
  for (int64_t i = int64_t(blockIdx.x) * kTile + tid; i < a.n; i += gstride)
    a.out[i] = load_cg(a.work + i);
  const int64_t nrep = int64_t(rounds_run) * a.nshards;
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < nrep; j += gstride) {
    const long long* src = reinterpret_cast<const long long*>(a.rep + j);
    long long* dst = reinterpret_cast<long long*>(a.rep_out + j);
#pragma unroll
    for (int q = 0; q < int(sizeof(yatt_round_report) / 8); ++q) dst[q] = __ldcg(src + q);
  }
  const int64_t nslot = int64_t(rounds_run) * a.slots;
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < nslot; j += gstride) {
    const int64_t ri = j / a.slots, k = j - ri * a.slots;
    const int s = last_le(a.mb_off, a.nshards, k);
    const int64_t q = k - __ldg(a.mb_off + s);
    const int64_t pr = ri * a.nshards + s;
    if (q < __ldcg(&a.rep[pr].num_microbatches)) {
      const long long* src = reinterpret_cast<const long long*>(a.mbs + j);
      long long* dst = reinterpret_cast<long long*>(a.mbs_out + __ldcg(a.pair_base + pr) + q);
      dst[0] = __ldcg(src);
      dst[1] = __ldcg(src + 1);
      dst[2] = __ldcg(src + 2);
    }
  }
  const unsigned ties = __ldcg(a.bar + 1);
  for (int64_t j = int64_t(blockIdx.x) * kTile + tid; j < min(int64_t(ties), int64_t(kTieCap));
       j += gstride)
    a.tie_out[j] = __ldcg(a.tie_key + j);
  if (blockIdx.x == 0 && tid == 0) {
    a.status[0] = rounds_run;
    a.status[1] = cursor;
    a.status[2] = ties;
  }
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

}  // namespace
}  // namespace yattb

using namespace yattb;

struct yatt_rounds {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  HostBuf stage;   // [tables | samples] packed by the caller, one H2D copy
  HostBuf outs;    // mapped outputs of one launch
  DevBuf dev;      // device copy of stage + scratch
  DevBuf ovr_dev;  // glibc overrides of uncertified draws (separate: may grow between re-runs)
  int grid_cap = 0;
  // accumulated over the launches of one call
  std::vector<yatt_round_report> reps;
  std::vector<yatt_mb_agg> mbs;
  std::vector<int32_t> first_lens;
  int64_t n = 0, redrawn = 0;
  int32_t rounds = 0, nshards = 0;
  const yatt_sample* final_samples = nullptr;
};

namespace {

// Host-side layout of the staging buffer: int64 shard_off[nshards+1],
// tile_off[nshards+1], mb_off[nshards] (aligned), then the samples.
size_t tables_bytes(int32_t nshards) { return align_up(sizeof(int64_t) * (3 * size_t(nshards) + 2)); }

}  // namespace

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

int yatt_rounds_stage(yatt_rounds_t h, int64_t n, int32_t nshards, yatt_sample** h_samples) {
  YATT_REQUIRE(h != nullptr && h_samples != nullptr, YATT_ERR_CONFIG, "rounds_stage: null argument");
  YATT_REQUIRE(n >= 0 && nshards >= 1, YATT_ERR_CONFIG, "rounds_stage: bad sizes");
  int rc = h->stage.reserve(tables_bytes(nshards) + sizeof(yatt_sample) * size_t(n));
  if (rc) return rc;
  *h_samples = reinterpret_cast<yatt_sample*>(static_cast<char*>(h->stage.h) + tables_bytes(nshards));
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
  YATT_REQUIRE(h->stage.bytes >= tables_bytes(nshards) + sizeof(yatt_sample) * size_t(n),
               YATT_ERR_CONFIG, "rounds_run: call yatt_rounds_stage first");
  YATT_REQUIRE(h_shard_offsets[0] == 0 && h_shard_offsets[nshards] == n, YATT_ERR_CONFIG,
               "rounds_run: shard offsets must span [0, n)");
  int dev_now = 0;
  YATT_TRY_CUDA(cudaGetDevice(&dev_now));
  YATT_REQUIRE(dev_now == h->device, YATT_ERR_CONFIG, "rounds_run: handle belongs to device %d",
               h->device);
  cudaStream_t st = stream ? as_stream(stream) : h->own_stream;

  // shard tables into the staging head
  int64_t* tab = static_cast<int64_t*>(h->stage.h);
  int64_t* t_shard = tab;
  int64_t* t_tile = tab + nshards + 1;
  int64_t* t_mb = tab + 2 * (nshards + 1);
  int64_t ntiles = 0, slots = 0;
  for (int32_t s = 0; s < nshards; ++s) {
    const int64_t sz = h_shard_offsets[s + 1] - h_shard_offsets[s];
    YATT_REQUIRE(sz >= 0, YATT_ERR_CONFIG, "shard offsets must ascend");
    t_shard[s] = h_shard_offsets[s];
    t_tile[s] = ntiles;
    t_mb[s] = slots;
    ntiles += ceil_div(sz, kTile);
    slots += ceil_div(sz, prm->microbatch_size);
  }
  t_shard[nshards] = n;
  t_tile[nshards] = ntiles;
  YATT_REQUIRE(n < (int64_t(1) << 40), YATT_ERR_CONFIG, "rounds_run: too many samples");

  const int32_t limit = round_limit > 0 ? round_limit : INT32_MAX;
  const int32_t K = std::min(kRoundsPerLaunch, limit);
  const size_t tb = tables_bytes(nshards), sb = sizeof(yatt_sample) * size_t(n);
  // device: [stage copy | work | tile_cnt | rep | mbs | pair_base | bar | ties | ovr keys | ovr lens]
  const size_t o_work = align_up(tb + sb);
  const size_t o_tile = o_work + align_up(sb);
  const size_t o_rep = o_tile + align_up(sizeof(int32_t) * size_t(ntiles));
  const size_t o_mbs = o_rep + align_up(sizeof(yatt_round_report) * size_t(K) * nshards);
  const size_t o_pair = o_mbs + align_up(sizeof(yatt_mb_agg) * size_t(K) * size_t(slots));
  const size_t o_bar = o_pair + align_up(sizeof(int64_t) * size_t(K) * nshards);
  const size_t o_ties = o_bar + 256;
  const size_t o_end = o_ties + align_up(sizeof(uint64_t) * kTieCap);
  // outputs (mapped): [samples | first_lens | reps | mbs | ties | status]
  const size_t p_first = align_up(sb);
  const size_t p_rep = p_first + align_up(sizeof(int32_t) * size_t(n));
  const size_t p_mbs = p_rep + align_up(sizeof(yatt_round_report) * size_t(K) * nshards);
  const size_t p_ties = p_mbs + align_up(sizeof(yatt_mb_agg) * size_t(K) * size_t(slots));
  const size_t p_status = p_ties + align_up(sizeof(uint64_t) * kTieCap);
  int rc = h->outs.reserve(p_status + 256);
  if (rc) return rc;

  h->reps.clear();
  h->mbs.clear();
  h->first_lens.clear();
  h->n = n;
  h->nshards = nshards;
  h->rounds = 0;
  h->redrawn = 0;
  const yatt_sample* h_in = reinterpret_cast<const yatt_sample*>(static_cast<char*>(h->stage.h) + tb);
  std::map<uint64_t, int32_t> ovr;  // (round << 40 | index) -> glibc length
  int32_t round = first_round;
  bool first_launch = true;
  bool stage_in = true;  // next launch's input: the host stage (else already on the device)
  char* ob = static_cast<char*>(h->outs.h);
  char* od = static_cast<char*>(h->outs.d);

  while (true) {
    if (stage_in) {
      rc = h->dev.reserve(o_end);
      if (rc) return rc;
    }
    const size_t ovr_bytes = align_up(sizeof(uint64_t) * ovr.size()) + align_up(sizeof(int32_t) * ovr.size());
    rc = h->ovr_dev.reserve(ovr_bytes);
    if (rc) return rc;
    char* db = static_cast<char*>(h->dev.p);
    char* dov = static_cast<char*>(h->ovr_dev.p);
    if (stage_in) {  // a re-run after host re-draws reuses the input on the device
      YATT_TRY_CUDA(cudaMemcpyAsync(db, h->stage.h, tb + sb, cudaMemcpyHostToDevice, st));
      stage_in = false;
    }
    if (!ovr.empty()) {
      std::vector<uint64_t> k;
      std::vector<int32_t> v;
      for (const auto& kv : ovr) {
        k.push_back(kv.first);
        v.push_back(kv.second);
      }
      YATT_TRY_CUDA(cudaMemcpyAsync(dov, k.data(), 8 * k.size(), cudaMemcpyHostToDevice, st));
      YATT_TRY_CUDA(cudaMemcpyAsync(dov + align_up(8 * k.size()), v.data(), 4 * v.size(),
                                    cudaMemcpyHostToDevice, st));
      YATT_TRY_CUDA(cudaStreamSynchronize(st));  // k, v are stack-owned
    }
    YATT_TRY_CUDA(cudaMemsetAsync(db + o_bar, 0, 8, st));
    RoundsArgs a{};
    a.in = reinterpret_cast<const yatt_sample*>(db + tb);
    a.work = reinterpret_cast<yatt_sample*>(db + o_work);
    a.out = reinterpret_cast<yatt_sample*>(od);
    a.first_lens = (want_first_lens && first_launch) ? reinterpret_cast<int32_t*>(od + p_first) : nullptr;
    a.shard_off = reinterpret_cast<const int64_t*>(db);
    a.tile_off = a.shard_off + nshards + 1;
    a.mb_off = a.shard_off + 2 * (nshards + 1);
    a.n = n;
    a.ntiles = ntiles;
    a.slots = slots;
    a.nshards = nshards;
    a.first_rank = first_rank;
    a.step = uint64_t(int64_t(step_index));
    a.first_round = round;
    a.round_limit = std::min<int64_t>(K, int64_t(limit) - (round - first_round));
    a.prm = *prm;
    a.band = g_tie_band;
    a.tile_cnt = reinterpret_cast<int32_t*>(db + o_tile);
    a.rep = reinterpret_cast<yatt_round_report*>(db + o_rep);
    a.mbs = reinterpret_cast<yatt_mb_agg*>(db + o_mbs);
    a.pair_base = reinterpret_cast<int64_t*>(db + o_pair);
    a.bar = reinterpret_cast<unsigned*>(db + o_bar);
    a.tie_key = reinterpret_cast<uint64_t*>(db + o_ties);
    a.ovr_key = reinterpret_cast<const uint64_t*>(dov);
    a.ovr_len = reinterpret_cast<const int32_t*>(dov + align_up(8 * ovr.size()));
    a.n_ovr = int32_t(ovr.size());
    a.rep_out = reinterpret_cast<yatt_round_report*>(od + p_rep);
    a.mbs_out = reinterpret_cast<yatt_mb_agg*>(od + p_mbs);
    a.tie_out = reinterpret_cast<uint64_t*>(od + p_ties);
    a.status = reinterpret_cast<int64_t*>(od + p_status);
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ntiles, h->grid_cap)));
    void* args[] = {&a};
    YATT_TRY_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(rollout_rounds_kernel),
                                              dim3(grid), dim3(kTile), args, 0, st));
    YATT_TRY_CUDA(cudaStreamSynchronize(st));
    const int64_t* status = reinterpret_cast<const int64_t*>(ob + p_status);
    const int64_t ties = status[2];
    if (ties > 0) {  // redo the uncertified draws with glibc and re-run this launch
      const uint64_t* keys = reinterpret_cast<const uint64_t*>(ob + p_ties);
      for (int64_t j = 0; j < std::min<int64_t>(ties, kTieCap); ++j) {
        const uint64_t key = keys[j];
        const int64_t idx = int64_t(key & ((uint64_t(1) << 40) - 1));
        const uint64_t rr = key >> 40;
        ovr[key] = length_keyed_glibc(prm->out_dist, prm->seed, kOutputLenStream,
                                      uint64_t(int64_t(step_index)), rr, h_in[idx].sample_id);
      }
      h->redrawn = int64_t(ovr.size());
      continue;
    }
    const int32_t rr = int32_t(status[0]);
    const int64_t nm = status[1];
    const auto* rp = reinterpret_cast<const yatt_round_report*>(ob + p_rep);
    h->reps.insert(h->reps.end(), rp, rp + int64_t(rr) * nshards);
    const auto* mp = reinterpret_cast<const yatt_mb_agg*>(ob + p_mbs);
    h->mbs.insert(h->mbs.end(), mp, mp + nm);
    if (a.first_lens) {
      const auto* fl = reinterpret_cast<const int32_t*>(ob + p_first);
      h->first_lens.assign(fl, fl + n);
    }
    h->rounds += rr;
    round += rr;
    first_launch = false;
    bool more = false;
    for (int32_t s = 0; s < nshards; ++s) more |= rp[int64_t(rr - 1) * nshards + s].pending_count > 0;
    if (!more || round - first_round >= limit) break;
    // continue from this launch's final state (the kernel never writes `in`)
    YATT_TRY_CUDA(cudaMemcpyAsync(db + tb, db + o_work, sb, cudaMemcpyDeviceToDevice, st));
  }
  h->final_samples = reinterpret_cast<const yatt_sample*>(ob);
  return YATT_OK;
}

int yatt_rounds_result(yatt_rounds_t h, yatt_rounds_view* v) {
  YATT_REQUIRE(h != nullptr && v != nullptr, YATT_ERR_CONFIG, "rounds_result: null argument");
  v->samples = h->final_samples;
  v->n_samples = h->n;
  v->first_round_lens = h->first_lens.empty() ? nullptr : h->first_lens.data();
  v->reports = h->reps.data();
  v->rounds = h->rounds;
  v->num_shards = h->nshards;
  v->microbatches = h->mbs.data();
  v->num_microbatches = int64_t(h->mbs.size());
  v->redrawn_on_host = h->redrawn;
  return YATT_OK;
}

int yatt_set_tie_band(double band) {
  YATT_REQUIRE(band >= 0 && band < 0.5, YATT_ERR_CONFIG, "tie band must lie in [0, 0.5)");
  g_tie_band = band;
  return YATT_OK;
}

}  // extern "C"
