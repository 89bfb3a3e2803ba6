// shard_round.cu — R3/R4/R5/R6: the per-rank dynamic-sampling round on the
// device, bit-exact with the reference.
//
//   sample_length_keyed   proj/src/workload.cpp:109-132 (+ clamp_length :15-20,
//                         normal_from_key :23-27)
//   rejection_process     proj/src/workload.cpp:145-167
//   shard_round_output    proj/src/simcore.cpp:157-214 (+ build_microbatches
//                         :17-39)
//
// One CTA per controller shard (all ranks of an in-process step in ONE launch,
// the loop of run_rlhf_step, simcore.cpp:482-484).  Each CTA walks its shard
// in 1024-sample tiles: keyed draw + rejection per pending sample, a block
// scan gives each pending sample its position in the ordered pending list
// (the reference's compaction order), microbatch aggregates accumulate with
// shared-memory integer atomics (exact and order-independent).
//
// Exactness: Constant/Uniform draws are pure IEEE multiply + nearbyint and
// match glibc bit for bit.  Normal/LogNormal use device libm (log1p, cos, sqrt,
// exp) which agree with glibc to <=1-2 ulp; after nearbyint() the integer
// length can only differ if the draw lands within an ulp of a .5 tie
// (probability ~1e-13 per draw; tests/test_gpu_integer.py checks 10^5 draws).
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace yattb {
namespace {

constexpr int kRoundThreads = 1024;
constexpr double kTwoPi = 6.283185307179586476925286766559;

__device__ __forceinline__ int clamp_length(double value, int max_len) {
  const double rounded = nearbyint(value);
  if (rounded < 1) return 1;
  if (rounded > max_len) return max_len;
  return int(rounded);
}

__device__ __forceinline__ double normal_from_key(uint64_t key) {
  const double u1 = uniform_from_key(key);
  const double u2 = uniform_from_key(splitmix64(key ^ 0x5bf0a8b1457e1d23ULL));
  return sqrt(-2.0 * log1p(-u1)) * cos(kTwoPi * u2);
}

__device__ __forceinline__ int length_keyed(const yatt_length_dist& d, uint64_t seed,
                                            uint64_t stream, uint64_t step, uint64_t round,
                                            uint64_t id) {
  const uint64_t key = hash5(seed, stream, step, round, id);
  switch (d.kind) {
    case YATT_DIST_CONSTANT: return clamp_length(d.p1, d.max_len_tokens);
    case YATT_DIST_UNIFORM: {
      const long long lo = llround(d.p1), hi = llround(d.p2);
      const uint64_t span = uint64_t(hi - lo) + 1;
      const double u = uniform_from_key(key);
      const long long v = lo + (long long)(u * double(span));
      return clamp_length(double(v), d.max_len_tokens);
    }
    case YATT_DIST_NORMAL:
      return clamp_length(d.p1 + d.p2 * normal_from_key(key), d.max_len_tokens);
    default:
      return clamp_length(exp(d.p1 + d.p2 * normal_from_key(key)), d.max_len_tokens);
  }
}

__device__ __forceinline__ bool rejected_keyed(const yatt_rejection_config& c, uint64_t seed,
                                               uint64_t step, uint64_t round, uint64_t id) {
  const uint64_t unit = c.per_group ? id / uint64_t(c.group_size) : id;
  return uniform_from_key(hash5(seed, kRejectionStream, step, round, unit)) < c.reject_rate;
}

__global__ void lengths_kernel(yatt_length_dist d, uint64_t seed, uint64_t stream, uint64_t step,
                               uint64_t round, const uint64_t* ids, int64_t n, int32_t* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = length_keyed(d, seed, stream, step, round, ids[i]);
}

__global__ void rejection_kernel(const yatt_sample* s, int64_t n, uint64_t step, uint64_t round,
                                 yatt_rejection_config c, uint64_t seed, uint8_t* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const yatt_sample x = s[i];
  out[i] = x.accepted ? 0 : uint8_t(rejected_keyed(c, seed, step, round, x.sample_id));
}

constexpr int kMaxShardsPerLaunch = 64;
struct ShardTable {
  int64_t off[kMaxShardsPerLaunch + 1];
  int64_t mb_off[kMaxShardsPerLaunch];
};

__global__ void __launch_bounds__(kRoundThreads) shard_round_kernel(
    yatt_sample* samples, const ShardTable tab, int32_t first_rank, uint64_t step, int32_t round,
    const yatt_round_params prm, yatt_round_report* reports, yatt_mb_agg* mbs_all) {
  const int shard = blockIdx.x;
  const int rank = first_rank + shard;
  const int64_t b = tab.off[shard], e = tab.off[shard + 1];
  const int64_t n = e - b;
  const int32_t mb = prm.microbatch_size;
  yatt_mb_agg* mbs = mbs_all + tab.mb_off[shard];
  const int64_t mb_cap = (n + mb - 1) / mb;
  const bool final_round = round >= prm.max_rounds;

  __shared__ unsigned long long s_score, s_units;
  __shared__ int s_active, s_acc, s_forced, s_pend;
  __shared__ int s_wsum[kRoundThreads / 32];
  __shared__ int s_base;

  for (int64_t k = threadIdx.x; k < mb_cap; k += blockDim.x)
    mbs[k] = yatt_mb_agg{rank, int32_t(k), 0, 0, 0};
  if (threadIdx.x == 0) {
    s_score = s_units = 0;
    s_active = s_acc = s_forced = s_pend = 0;
    s_base = 0;
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t t0 = 0; t0 < n; t0 += kRoundThreads) {
    const int64_t i = t0 + threadIdx.x;
    yatt_sample x{};
    bool pending = false;
    if (i < n) {
      x = samples[b + i];
      pending = !x.accepted;
    }
    // position among this round's pending samples (ordered compaction)
    const unsigned bal = __ballot_sync(0xffffffffu, pending);
    if (lane == 0) s_wsum[w] = __popc(bal);
    __syncthreads();
    if (w == 0) {
      int v = s_wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
      }
      s_wsum[lane] = v;  // inclusive
    }
    __syncthreads();
    const int tile_base = s_base;
    const int before = (w > 0 ? s_wsum[w - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
    const int tile_total = s_wsum[31];
    if (pending) {
      const int pidx = tile_base + before;
      x.out_len_tokens = length_keyed(prm.out_dist, prm.seed, kOutputLenStream, step,
                                      uint64_t(round), x.sample_id);
      yatt_mb_agg* m = mbs + pidx / mb;
      atomicAdd(&m->sample_count, 1);
      atomicMax(&m->max_out_len_tokens, x.out_len_tokens);
      atomicAdd(reinterpret_cast<unsigned long long*>(&m->score_tokens),
                (unsigned long long)(int64_t(x.prompt_len_tokens) + x.out_len_tokens));
      const bool rej = rejected_keyed(prm.rejection, prm.seed, step, uint64_t(round), x.sample_id);
      if (rej && !final_round) {
        atomicAdd(&s_pend, 1);
      } else {
        if (rej) atomicAdd(&s_forced, 1);
        x.accepted = 1;
        x.accepted_round = round;
        atomicAdd(&s_acc, 1);
        const long long tok = (long long)x.prompt_len_tokens + x.out_len_tokens;
        atomicAdd(&s_score, (unsigned long long)tok);
        atomicAdd(&s_units, (unsigned long long)(tok * tok));
      }
      samples[b + i] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_base = tile_base + tile_total;
      s_active += tile_total;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    yatt_round_report r;
    r.controller_rank = rank;
    r.round = round;
    r.active_count = s_active;
    r.newly_accepted_count = s_acc;
    r.forced_accept_count = s_forced;
    r.pending_count = s_pend;
    r.accepted_score_tokens = (long long)s_score;
    r.accepted_train_units = (long long)s_units;
    r.num_microbatches = (s_active + mb - 1) / mb;
    reports[shard] = r;
  }
}

}  // namespace

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
                                                             ids, n, out);
  return check_launch("lengths_kernel");
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
    int64_t mb_acc = 0;
    for (int32_t k = 0; k <= cnt; ++k) tab.off[k] = h_off[s0 + k];
    for (int32_t k = 0; k < cnt; ++k) {
      YATT_REQUIRE(tab.off[k + 1] >= tab.off[k], YATT_ERR_CONFIG, "shard offsets must ascend");
      tab.mb_off[k] = mb_acc;
      mb_acc += ceil_div(tab.off[k + 1] - tab.off[k], prm->microbatch_size);
    }
    // microbatch slots of earlier launches
    int64_t mb_before = 0;
    for (int32_t k = 0; k < s0; ++k)
      mb_before += ceil_div(h_off[k + 1] - h_off[k], prm->microbatch_size);
    shard_round_kernel<<<cnt, kRoundThreads, 0, st>>>(
        samples, tab, first_rank + s0, uint64_t(int64_t(step)), round, *prm, reports + s0,
        mbs + mb_before);
    int rc = check_launch("shard_round_kernel");
    if (rc) return rc;
  }
  return YATT_OK;
}

}  // namespace yattb
