// shard_round.cu — R3/R4/R5/R6: the per-rank dynamic-sampling round on the
// device, bit-exact with the reference.
//
//   sample_length_keyed   proj/src/workload.cpp:109-132 (+ clamp_length :15-20,
//                         normal_from_key :23-27)
//   rejection_process     proj/src/workload.cpp:145-167
//   shard_round_output    proj/src/simcore.cpp:157-214 (+ build_microbatches
//                         :17-39)
//
// All controller shards of an in-process step are processed by one set of
// launches (the loop of run_rlhf_step, simcore.cpp:482-484), one CTA per
// 256-sample tile of any shard: keyed draw + rejection per pending sample, a
// ballot scan plus the pending count of the earlier tiles gives each pending
// sample its position in the ordered pending list (the reference's
// compaction order), microbatch aggregates and report counters accumulate
// with integer atomics (exact and order-independent).
//
// Exactness (keyed_draw.cuh): Constant/Uniform draws are pure IEEE multiply +
// nearbyint and match glibc bit for bit.  Normal/LogNormal draws are
// certified: a draw within 1e-9 relative of a .5 rounding tie is not trusted.
// The host-facing entry points (lengths_host here, rollout_rounds.cu) redo
// those with glibc; these device-resident ones count them in g_uncertified
// (yatt_uncertified_draws) so a caller can detect the ~1e-9-per-draw event.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "keyed_draw.cuh"

namespace yattb {
namespace {


// Draws of the device-resident entry points not certified equal to glibc's
// (keyed_draw.cuh); read and reset by yatt_uncertified_draws.
__device__ unsigned long long g_uncertified = 0;

__device__ __forceinline__ int length_keyed(const yatt_length_dist& d, uint64_t seed,
                                            uint64_t stream, uint64_t step, uint64_t round,
                                            uint64_t id, double band) {
  bool tie = false;
  const int len = length_keyed_dev(d, seed, stream, step, round, id, band, &tie);
  if (tie) atomicAdd(&g_uncertified, 1ull);
  return len;
}

__device__ __forceinline__ bool rejected_keyed(const yatt_rejection_config& c, uint64_t seed,
                                               uint64_t step, uint64_t round, uint64_t id) {
  const uint64_t unit = c.per_group ? id / uint64_t(c.group_size) : id;
  return uniform_from_key(hash5(seed, kRejectionStream, step, round, unit)) < c.reject_rate;
}

__global__ void lengths_kernel(yatt_length_dist d, uint64_t seed, uint64_t stream, uint64_t step,
                               uint64_t round, const uint64_t* ids, int64_t n, int32_t* out,
                               double band) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = length_keyed(d, seed, stream, step, round, ids[i], band);
}

// Host-facing variant: uncertified draws are listed (index) for a glibc redo.
__global__ void lengths_cert_kernel(yatt_length_dist d, uint64_t seed, uint64_t stream,
                                    uint64_t step, uint64_t round, const uint64_t* ids, int64_t n,
                                    int32_t* out, double band, unsigned long long* cnt,
                                    int64_t* list, int64_t cap) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool tie = false;
  out[i] = length_keyed_dev(d, seed, stream, step, round, ids[i], band, &tie);
  if (tie) {
    const unsigned long long k = atomicAdd(cnt, 1ull);
    if (k < (unsigned long long)cap) list[k] = i;
  }
}

__global__ void rejection_kernel(const yatt_sample* s, int64_t n, uint64_t step, uint64_t round,
                                 yatt_rejection_config c, uint64_t seed, uint8_t* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const yatt_sample x = s[i];
  out[i] = x.accepted ? 0 : uint8_t(rejected_keyed(c, seed, step, round, x.sample_id));
}

constexpr int kMaxShardsPerLaunch = 64;

// Three stream-ordered launches per round (all shards at once):
//   init     : zero every shard's report and microbatch slots
//   tile     : one CTA per 256-sample tile of any shard (the whole GPU works
//              on a 16K-sample round); the tile's first pending index is the
//              count of pending samples earlier in its shard (input state,
//              independent of this round's draws), the in-tile order comes
//              from a ballot/warp scan; results accumulate with integer
//              atomics (exact, order-free)
//   finalize : num_microbatches = ceil(active / microbatch_size)
constexpr int kTileSamples = 256;
// Transient `accepted` value of samples accepted by the running launch: other
// CTAs still count them as pending-at-round-start (race-free tile bases).
constexpr int32_t kAcceptedThisRound = 0x7f000001;
__device__ __forceinline__ int pending_at_start(int32_t a) {
  return (a == 0 || a == kAcceptedThisRound) ? 1 : 0;
}
struct ShardTable {
  int64_t off[kMaxShardsPerLaunch + 1];
  int64_t mb_off[kMaxShardsPerLaunch];
  int64_t tile_off[kMaxShardsPerLaunch + 1];
  int32_t nshards;
};

__global__ void shard_round_init_kernel(const ShardTable tab, int32_t first_rank, int32_t round,
                                        int32_t mb, yatt_round_report* reports,
                                        yatt_mb_agg* mbs_all) {
  const int shard = blockIdx.x;
  const int rank = first_rank + shard;
  const int64_t n = tab.off[shard + 1] - tab.off[shard];
  yatt_mb_agg* mbs = mbs_all + tab.mb_off[shard];
  for (int64_t k = threadIdx.x; k < (n + mb - 1) / mb; k += blockDim.x)
    mbs[k] = yatt_mb_agg{rank, int32_t(k), 0, 0, 0};
  if (threadIdx.x == 0) reports[shard] = yatt_round_report{rank, round, 0, 0, 0, 0, 0, 0, 0};
}

__global__ void __launch_bounds__(kTileSamples) shard_round_tile_kernel(
    yatt_sample* samples, const ShardTable tab, uint64_t step, int32_t round,
    const yatt_round_params prm, yatt_round_report* reports, yatt_mb_agg* mbs_all, double band) {
  int shard = 0;
  while (shard + 1 < tab.nshards && tab.tile_off[shard + 1] <= blockIdx.x) ++shard;
  const int64_t b = tab.off[shard], e = tab.off[shard + 1];
  const int64_t t0 = b + (int64_t(blockIdx.x) - tab.tile_off[shard]) * kTileSamples;
  const int32_t mb = prm.microbatch_size;
  yatt_mb_agg* mbs = mbs_all + tab.mb_off[shard];
  yatt_round_report* rep = reports + shard;
  const bool final_round = round >= prm.max_rounds;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ int s_wsum[kTileSamples / 32];
  __shared__ int s_before;

  // pending samples of this shard before the tile
  int cnt = 0;
  for (int64_t i = b + threadIdx.x; i < t0; i += kTileSamples) cnt += pending_at_start(samples[i].accepted);
  cnt = warp_sum(cnt);
  if (lane == 0) s_wsum[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int k = 0; k < kTileSamples / 32; ++k) s += s_wsum[k];
    s_before = s;
  }
  __syncthreads();

  const int64_t i = t0 + threadIdx.x;
  yatt_sample x{};
  bool pending = false;
  if (i < e) {
    x = samples[i];
    pending = x.accepted == 0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, pending);
  if (lane == 0) s_wsum[w] = __popc(bal);
  __syncthreads();
  int before = s_before + __popc(bal & ((1u << lane) - 1u));
  for (int k = 0; k < w; ++k) before += s_wsum[k];
  int tile_pending = 0, acc = 0, forced = 0, pend = 0;
  unsigned long long score = 0, units = 0;
  if (pending) {
    tile_pending = 1;
    x.out_len_tokens = length_keyed(prm.out_dist, prm.seed, kOutputLenStream, step,
                                    uint64_t(round), x.sample_id, band);
    yatt_mb_agg* m = mbs + before / mb;
    atomicAdd(&m->sample_count, 1);
    atomicMax(&m->max_out_len_tokens, x.out_len_tokens);
    atomicAdd(reinterpret_cast<unsigned long long*>(&m->score_tokens),
              (unsigned long long)(int64_t(x.prompt_len_tokens) + x.out_len_tokens));
    const bool rej = rejected_keyed(prm.rejection, prm.seed, step, uint64_t(round), x.sample_id);
    if (rej && !final_round) {
      pend = 1;
    } else {
      forced = rej ? 1 : 0;
      x.accepted = kAcceptedThisRound;  // -> 1 in finalize
      x.accepted_round = round;
      acc = 1;
      const long long tok = (long long)x.prompt_len_tokens + x.out_len_tokens;
      score = (unsigned long long)tok;
      units = (unsigned long long)(tok * tok);
    }
    samples[i] = x;
  }
  // warp-aggregate, then one atomic per warp per field
  tile_pending = warp_sum(tile_pending);
  acc = warp_sum(acc);
  forced = warp_sum(forced);
  pend = warp_sum(pend);
  score = warp_sum(score);
  units = warp_sum(units);
  if (lane == 0 && tile_pending) {
    atomicAdd(&rep->active_count, tile_pending);
    atomicAdd(&rep->newly_accepted_count, acc);
    atomicAdd(&rep->forced_accept_count, forced);
    atomicAdd(&rep->pending_count, pend);
    atomicAdd(reinterpret_cast<unsigned long long*>(&rep->accepted_score_tokens), score);
    atomicAdd(reinterpret_cast<unsigned long long*>(&rep->accepted_train_units), units);
  }
}

__global__ void shard_round_finalize_kernel(int32_t nshards, int32_t mb, yatt_sample* samples,
                                            int64_t lo, int64_t hi,
                                            yatt_round_report* reports) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nshards) reports[s].num_microbatches = (reports[s].active_count + mb - 1) / mb;
  for (int64_t i = lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < hi;
       i += int64_t(gridDim.x) * blockDim.x)
    if (samples[i].accepted == kAcceptedThisRound) samples[i].accepted = 1;
}

// One warp: sums of the reports' integer fields (order-free, exact).
__global__ void reduce_reports_kernel(const yatt_round_report* r, int32_t n, int64_t* out) {
  long long a = 0, p = 0, f = 0, u = 0, sc = 0;
  for (int i = threadIdx.x; i < n; i += 32) {
    a += r[i].active_count;
    p += r[i].pending_count;
    f += r[i].forced_accept_count;
    u += r[i].accepted_train_units;
    sc += r[i].accepted_score_tokens;
  }
  a = warp_sum(a);
  p = warp_sum(p);
  f = warp_sum(f);
  u = warp_sum(u);
  sc = warp_sum(sc);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = p;
    out[2] = f;
    out[3] = u;
    out[4] = sc;
    out[5] = p > 0 ? 1 : 0;
  }
}

}  // namespace

int reduce_reports_launch(const yatt_round_report* r, int32_t n, int64_t* out, cudaStream_t st) {
  YATT_REQUIRE(n >= 0 && out != nullptr, YATT_ERR_CONFIG, "reduce_round_reports: bad arguments");
  reduce_reports_kernel<<<1, 32, 0, st>>>(r, n, out);
  return check_launch("reduce_reports_kernel");
}

int validate_dist(const yatt_length_dist* d) {
  YATT_REQUIRE(d != nullptr, YATT_ERR_CONFIG, "null length distribution");
  YATT_REQUIRE(d->max_len_tokens >= 1, YATT_ERR_DISTRIBUTION, "max_len_tokens must be at least 1");
  switch (d->kind) {
    case YATT_DIST_CONSTANT:
      YATT_REQUIRE(d->p1 >= 1, YATT_ERR_DISTRIBUTION, "constant length must be at least 1");
      break;
    case YATT_DIST_UNIFORM:
      YATT_REQUIRE(d->p1 >= 1, YATT_ERR_DISTRIBUTION, "uniform low bound must be at least 1");
      YATT_REQUIRE(d->p2 >= d->p1, YATT_ERR_DISTRIBUTION, "uniform high bound below low bound");
      break;
    case YATT_DIST_NORMAL:
      YATT_REQUIRE(d->p2 >= 0, YATT_ERR_DISTRIBUTION, "normal stddev must be non-negative");
      break;
    case YATT_DIST_LOGNORMAL:
      YATT_REQUIRE(d->p2 >= 0, YATT_ERR_DISTRIBUTION, "lognormal sigma must be non-negative");
      break;
    default: return set_error(YATT_ERR_CONFIG, "unknown distribution kind value %d", d->kind);
  }
  return YATT_OK;
}

int validate_rejection(const yatt_rejection_config* c) {
  YATT_REQUIRE(c != nullptr, YATT_ERR_CONFIG, "null rejection config");
  YATT_REQUIRE(c->reject_rate >= 0 && c->reject_rate < 1, YATT_ERR_CONFIG,
               "reject_rate must lie in [0, 1)");
  YATT_REQUIRE(!c->per_group || c->group_size > 0, YATT_ERR_CONFIG,
               "group_size must be positive for per-group rejection");
  return YATT_OK;
}

int lengths_launch(const yatt_length_dist* d, uint64_t seed, uint64_t stream_id, uint64_t step,
                   uint64_t round, const uint64_t* ids, int64_t n, int32_t* out, cudaStream_t st) {
  YATT_REQUIRE(d != nullptr && d->kind >= 0 && d->kind <= 3, YATT_ERR_CONFIG,
               "unknown distribution kind value");
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "sample_lengths: n must be >= 0");
  if (n == 0) return YATT_OK;
  lengths_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(*d, seed, stream_id, step, round,
                                                             ids, n, out, tie_band());
  return check_launch("lengths_kernel");
}

int uncertified_draws(int64_t* count, int32_t reset) {
  YATT_REQUIRE(count != nullptr, YATT_ERR_CONFIG, "uncertified_draws: null count");
  YATT_TRY_CUDA(cudaDeviceSynchronize());
  unsigned long long v = 0;
  YATT_TRY_CUDA(cudaMemcpyFromSymbol(&v, g_uncertified, sizeof(v)));
  *count = int64_t(v);
  if (reset) {
    const unsigned long long z = 0;
    YATT_TRY_CUDA(cudaMemcpyToSymbol(g_uncertified, &z, sizeof(z)));
  }
  return YATT_OK;
}

// Host ids -> host lengths, bit-exact for every kind: device draws, then the
// uncertified ones (keyed_draw.cuh) redone with glibc.
int lengths_host(const yatt_length_dist* d, uint64_t seed, uint64_t stream_id, uint64_t step,
                 uint64_t round, const uint64_t* h_ids, int64_t n, int32_t* h_out) {
  int rc = validate_dist(d);
  if (rc) return rc;
  YATT_REQUIRE(n >= 0 && (n == 0 || (h_ids && h_out)), YATT_ERR_CONFIG,
               "sample_lengths: bad arguments");
  if (n == 0) return YATT_OK;
  constexpr int64_t kCap = 4096;
  char* buf = nullptr;
  const size_t bytes = size_t(n) * 12 + 8 + kCap * 8;
  YATT_TRY_CUDA(cudaMalloc(&buf, bytes));
  uint64_t* ids = reinterpret_cast<uint64_t*>(buf);
  int32_t* out = reinterpret_cast<int32_t*>(buf + size_t(n) * 8);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(buf + ((size_t(n) * 12 + 7) & ~size_t(7)));
  int64_t* list = reinterpret_cast<int64_t*>(cnt + 1);
  unsigned long long h_cnt = 0;
  std::vector<int64_t> h_list;
  cudaError_t e = cudaMemcpy(ids, h_ids, size_t(n) * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(cnt, 0, 8);
  if (e == cudaSuccess) {
    lengths_cert_kernel<<<unsigned(ceil_div(n, 256)), 256>>>(*d, seed, stream_id, step, round, ids,
                                                             n, out, tie_band(), cnt, list, kCap);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(h_out, out, size_t(n) * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&h_cnt, cnt, 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && h_cnt > 0 && h_cnt <= (unsigned long long)kCap) {
    h_list.resize(size_t(h_cnt));
    e = cudaMemcpy(h_list.data(), list, size_t(h_cnt) * 8, cudaMemcpyDeviceToHost);
  }
  cudaFree(buf);
  if (e != cudaSuccess) return set_error(YATT_ERR_CUDA, "sample_lengths: %s", cudaGetErrorString(e));
  if (h_cnt > (unsigned long long)kCap) {  // (only with a widened band) redo all on the host
    for (int64_t i = 0; i < n; ++i)
      h_out[i] = length_keyed_glibc(*d, seed, stream_id, step, round, h_ids[i]);
  } else {
    for (int64_t i : h_list) h_out[i] = length_keyed_glibc(*d, seed, stream_id, step, round, h_ids[i]);
  }
  return YATT_OK;
}

int rejection_launch(const yatt_sample* s, int64_t n, int32_t step, int32_t round,
                     const yatt_rejection_config* c, uint64_t seed, uint8_t* out,
                     cudaStream_t st) {
  int rc = validate_rejection(c);
  if (rc) return rc;
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "rejection: n must be >= 0");
  if (n == 0) return YATT_OK;
  rejection_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(
      s, n, uint64_t(int64_t(step)), uint64_t(int64_t(round)), *c, seed, out);
  return check_launch("rejection_kernel");
}

int shard_round_launch(yatt_sample* samples, const int64_t* h_off, int32_t nshards,
                       int32_t first_rank, int32_t step, int32_t round,
                       const yatt_round_params* prm, yatt_round_report* reports, yatt_mb_agg* mbs,
                       cudaStream_t st) {
  YATT_REQUIRE(prm != nullptr, YATT_ERR_CONFIG, "shard_round: null params");
  YATT_REQUIRE(prm->microbatch_size > 0, YATT_ERR_CONFIG, "microbatch_size must be positive");
  YATT_REQUIRE(prm->out_dist.kind >= 0 && prm->out_dist.kind <= 3, YATT_ERR_CONFIG,
               "unknown distribution kind value");
  // rejection_process validation is not performed by the reference's inline
  // predicate (simcore.cpp:187-198); only group_size must be usable.
  YATT_REQUIRE(!prm->rejection.per_group || prm->rejection.group_size > 0, YATT_ERR_CONFIG,
               "group_size must be positive for per-group rejection");
  YATT_REQUIRE(nshards >= 0 && h_off != nullptr, YATT_ERR_CONFIG, "shard_round: bad shard table");
  for (int32_t s0 = 0; s0 < nshards; s0 += kMaxShardsPerLaunch) {
    const int32_t cnt = min(kMaxShardsPerLaunch, nshards - s0);
    ShardTable tab;
    tab.nshards = cnt;
    int64_t mb_acc = 0;
    tab.tile_off[0] = 0;
    for (int32_t k = 0; k <= cnt; ++k) tab.off[k] = h_off[s0 + k];
    for (int32_t k = 0; k < cnt; ++k) {
      YATT_REQUIRE(tab.off[k + 1] >= tab.off[k], YATT_ERR_CONFIG, "shard offsets must ascend");
      YATT_REQUIRE(tab.off[k + 1] - tab.off[k] < (int64_t(1) << 31), YATT_ERR_CONFIG,
                   "shard_round: shard too large");
      tab.mb_off[k] = mb_acc;
      mb_acc += ceil_div(tab.off[k + 1] - tab.off[k], prm->microbatch_size);
      tab.tile_off[k + 1] = tab.tile_off[k] + ceil_div(tab.off[k + 1] - tab.off[k], kTileSamples);
    }
    // microbatch slots of earlier launches
    int64_t mb_before = 0;
    for (int32_t k = 0; k < s0; ++k)
      mb_before += ceil_div(h_off[k + 1] - h_off[k], prm->microbatch_size);
    if (cnt == 0) continue;
    shard_round_init_kernel<<<cnt, 256, 0, st>>>(tab, first_rank + s0, round,
                                                 prm->microbatch_size, reports + s0,
                                                 mbs + mb_before);
    int rc = check_launch("shard_round_init_kernel");
    if (rc) return rc;
    if (tab.tile_off[cnt] > 0) {
      shard_round_tile_kernel<<<unsigned(tab.tile_off[cnt]), kTileSamples, 0, st>>>(
          samples, tab, uint64_t(int64_t(step)), round, *prm, reports + s0, mbs + mb_before,
          tie_band());
      rc = check_launch("shard_round_tile_kernel");
      if (rc) return rc;
    }
    shard_round_finalize_kernel<<<unsigned(max64(1, min64(ceil_div(tab.off[cnt] - tab.off[0], 256), 4 * num_sms()))), 256, 0, st>>>(
        cnt, prm->microbatch_size, samples, tab.off[0], tab.off[cnt], reports + s0);
    rc = check_launch("shard_round_finalize_kernel");
    if (rc) return rc;
  }
  return YATT_OK;
}

}  // namespace yattb
