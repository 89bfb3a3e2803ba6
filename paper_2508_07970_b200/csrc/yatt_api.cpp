// yatt_api.cpp — the drop-in C++ host API (include/yatt/*.hpp) over the C ABI.
//
// STL-typed entry points keep the reference's signatures and exception
// types; they own the H2D/D2H copies around the device kernels and block
// only because the reference API returns host data.  Device scratch is a
// per-thread grow-only arena (no allocation once warm).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "yatt/balancer.hpp"
#include "yatt/common.hpp"
#include "yatt/errors.hpp"
#include "yatt/experience.hpp"
#include "yatt/simcore.hpp"
#include "yatt/workload.hpp"
#include "yatt_cuda.h"

namespace yatt {

namespace detail {

void throw_status(int status) {
  if (status == YATT_OK) return;
  const std::string msg = yatt_last_error_message();
  switch (status) {
    case YATT_ERR_CONFIG:
    case YATT_ERR_WORKSPACE: throw ConfigError(msg);
    case YATT_ERR_RANK: throw RankOutOfRange(msg);
    case YATT_ERR_DISTRIBUTION: throw InvalidDistribution(msg);
    default: throw DeviceError(msg);
  }
}

namespace {

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Grow-only device scratch, one slot per use site.
struct Arena {
  void* ptr[8] = {};
  size_t cap[8] = {};
  void* get(int slot, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (bytes > cap[slot]) {
      if (ptr[slot]) cudaFree(ptr[slot]);
      ptr[slot] = nullptr;
      cap[slot] = 0;
      cuda_ok(cudaMalloc(&ptr[slot], bytes), "cudaMalloc");
      cap[slot] = bytes;
    }
    return ptr[slot];
  }
};
thread_local Arena g_arena;

template <typename T>
T* dev(int slot, size_t n) {
  return static_cast<T*>(g_arena.get(slot, n * sizeof(T)));
}

void h2d(void* d, const void* h, size_t bytes) {
  if (bytes) cuda_ok(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
}
void d2h(void* h, const void* d, size_t bytes) {
  if (bytes) cuda_ok(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
}

yatt_length_dist to_c(const workload::LengthDistribution& d) {
  return yatt_length_dist{static_cast<int32_t>(d.kind), d.max_len_tokens, d.p1, d.p2};
}
yatt_rejection_config to_c(const workload::RejectionConfig& c) {
  return yatt_rejection_config{c.reject_rate, c.per_group ? 1 : 0, c.group_size};
}

}  // namespace
}  // namespace detail

// ------------------------------------------------------------- common ----
std::string hex_encode(std::string_view bytes) {
  static const char* digits = "0123456789abcdef";
  std::string out;
  out.reserve(bytes.size() * 2);
  for (unsigned char c : bytes) {
    out.push_back(digits[c >> 4]);
    out.push_back(digits[c & 15]);
  }
  return out;
}

std::string hex_decode(std::string_view hex) {
  auto nib = [](char c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    throw ConfigError("invalid hex digit");
  };
  if (hex.size() % 2) throw ConfigError("hex string has odd length");
  std::string out(hex.size() / 2, '\0');
  for (size_t i = 0; i < out.size(); ++i)
    out[i] = static_cast<char>((nib(hex[2 * i]) << 4) | nib(hex[2 * i + 1]));
  return out;
}

// ----------------------------------------------------------- workload ----
namespace workload {

std::string dist_kind_name(DistKind kind) {
  switch (kind) {
    case DistKind::kConstant: return "constant";
    case DistKind::kUniform: return "uniform";
    case DistKind::kNormal: return "normal";
    case DistKind::kLogNormal: return "lognormal";
  }
  throw ConfigError("unknown distribution kind value");
}

DistKind dist_kind_from_name(const std::string& name) {
  for (DistKind k : {DistKind::kConstant, DistKind::kUniform, DistKind::kNormal,
                     DistKind::kLogNormal})
    if (dist_kind_name(k) == name) return k;
  throw ConfigError("unknown distribution kind: " + name);
}

void LengthDistribution::validate() const {
  const yatt_length_dist d = detail::to_c(*this);
  // Same checks as the device-side validator (shard_round.cu validate_dist).
  if (d.max_len_tokens < 1) throw InvalidDistribution("max_len_tokens must be at least 1");
  switch (kind) {
    case DistKind::kConstant:
      if (p1 < 1) throw InvalidDistribution("constant length must be at least 1");
      break;
    case DistKind::kUniform:
      if (p1 < 1) throw InvalidDistribution("uniform low bound must be at least 1");
      if (p2 < p1) throw InvalidDistribution("uniform high bound below low bound");
      break;
    case DistKind::kNormal:
      if (p2 < 0) throw InvalidDistribution("normal stddev must be non-negative");
      break;
    case DistKind::kLogNormal:
      if (p2 < 0) throw InvalidDistribution("lognormal sigma must be non-negative");
      break;
  }
}

double LengthDistribution::mean() const {
  switch (kind) {
    case DistKind::kConstant:
    case DistKind::kNormal: return p1;
    case DistKind::kUniform: return 0.5 * (p1 + p2);
    case DistKind::kLogNormal: return std::exp(p1 + 0.5 * p2 * p2);
  }
  throw ConfigError("unknown distribution kind value");
}

LengthDistribution LengthDistribution::scaled(double factor) const {
  LengthDistribution r = *this;
  if (kind == DistKind::kLogNormal) {
    r.p1 = p1 + std::log(factor);  // location shift in log space
  } else {
    r.p1 = p1 * factor;
    if (kind != DistKind::kConstant) r.p2 = p2 * factor;
  }
  return r;
}

namespace {
int clamp_to_length(double v, int max_len) {
  const double r = std::nearbyint(v);
  return r < 1 ? 1 : (r > max_len ? max_len : static_cast<int>(r));
}
double keyed_normal(std::uint64_t key) {
  const double u1 = uniform_from_key(key);
  const double u2 = uniform_from_key(splitmix64(key ^ 0x5bf0a8b1457e1d23ULL));
  return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(6.283185307179586476925286766559 * u2);
}
}  // namespace

int sample_length_keyed(const LengthDistribution& dist, std::uint64_t seed, std::uint64_t stream,
                        std::uint64_t step, std::uint64_t round, std::uint64_t sample_id) {
  const std::uint64_t key = hash_key({seed, stream, step, round, sample_id});
  switch (dist.kind) {
    case DistKind::kConstant: return clamp_to_length(dist.p1, dist.max_len_tokens);
    case DistKind::kUniform: {
      const long long lo = std::llround(dist.p1), hi = std::llround(dist.p2);
      const double span = static_cast<double>(static_cast<std::uint64_t>(hi - lo) + 1);
      return clamp_to_length(
          static_cast<double>(lo + static_cast<long long>(uniform_from_key(key) * span)),
          dist.max_len_tokens);
    }
    case DistKind::kNormal:
      return clamp_to_length(dist.p1 + dist.p2 * keyed_normal(key), dist.max_len_tokens);
    case DistKind::kLogNormal:
      return clamp_to_length(std::exp(dist.p1 + dist.p2 * keyed_normal(key)),
                             dist.max_len_tokens);
  }
  throw ConfigError("unknown distribution kind value");
}

std::vector<int> sample_lengths(const LengthDistribution& dist, int n, std::uint64_t seed) {
  if (n <= 0) return {};
  std::vector<std::uint64_t> ids(static_cast<size_t>(n));
  std::iota(ids.begin(), ids.end(), std::uint64_t{0});
  const yatt_length_dist d = detail::to_c(dist);
  std::vector<int> out(static_cast<size_t>(n));
  detail::throw_status(yatt_sample_lengths_host(&d, seed, kOutputLenStream, 0, 0, ids.data(), n,
                                                out.data()));
  return out;
}

std::vector<bool> rejection_process(const RolloutBatch& batch, int round,
                                    const RejectionConfig& config, std::uint64_t seed) {
  const size_t n = batch.samples.size();
  std::vector<yatt_sample> packed(n);
  for (size_t i = 0; i < n; ++i) {
    const RolloutSample& s = batch.samples[i];
    packed[i] = yatt_sample{s.sample_id, s.prompt_len_tokens, s.target_out_len_tokens,
                            s.accepted_round, s.accepted ? 1 : 0};
  }
  auto* d_s = detail::dev<yatt_sample>(0, n);
  auto* d_f = detail::dev<std::uint8_t>(1, n);
  detail::h2d(d_s, packed.data(), n * sizeof(yatt_sample));
  const yatt_rejection_config c = detail::to_c(config);
  detail::throw_status(yatt_rejection_flags(d_s, static_cast<std::int64_t>(n), batch.step_index,
                                            round, &c, seed, d_f, nullptr));
  std::vector<std::uint8_t> flags(n);
  detail::d2h(flags.data(), d_f, n);
  return std::vector<bool>(flags.begin(), flags.end());
}

LengthDistribution drift_schedule(int step, const LengthDistribution& base,
                                  double drift_rate_per_step) {
  if (drift_rate_per_step < 0) throw ConfigError("drift_rate_per_step must be non-negative");
  double factor = std::pow(1.0 + drift_rate_per_step, static_cast<double>(step));
  const double m = base.mean();
  if (m > 0) factor = std::min(factor, std::max(static_cast<double>(base.max_len_tokens) / m, 1.0));
  return base.scaled(factor);
}

ShardRange shard_dataset(std::uint64_t total, int num_controllers, int controller_rank) {
  ShardRange r;
  detail::throw_status(
      yatt_shard_dataset(total, num_controllers, controller_rank, &r.begin, &r.end));
  return r;
}

}  // namespace workload

// ------------------------------------------------------------- simcore ----
namespace sim {
namespace {

yatt_round_params to_c(const RoundParams& p) {
  return yatt_round_params{detail::to_c(p.out_dist), detail::to_c(p.rejection), p.seed,
                           p.microbatch_size, p.max_rounds};
}

ShardRoundReport from_c(const yatt_round_report& r, const yatt_mb_agg* mbs) {
  ShardRoundReport out;
  out.controller_rank = r.controller_rank;
  out.round = r.round;
  out.active_count = r.active_count;
  out.newly_accepted_count = r.newly_accepted_count;
  out.forced_accept_count = r.forced_accept_count;
  out.pending_count = r.pending_count;
  out.accepted_score_tokens = r.accepted_score_tokens;
  out.accepted_train_units = r.accepted_train_units;
  out.microbatches.reserve(static_cast<size_t>(r.num_microbatches));
  for (std::int64_t k = 0; k < r.num_microbatches; ++k)
    out.microbatches.push_back(MicrobatchAggregate{mbs[k].controller_rank, mbs[k].mb_index,
                                                   mbs[k].sample_count,
                                                   mbs[k].max_out_len_tokens,
                                                   mbs[k].score_tokens});
  return out;
}

std::int64_t mb_slots(std::int64_t n, int mb) { return mb > 0 ? (n + mb - 1) / mb : 0; }

}  // namespace

// One rounds engine per thread (rollout_rounds.cu): pinned mapped staging and
// device scratch, grow-only; the reference's functions are callable
// concurrently on distinct states.
struct RoundsHandle {
  yatt_rounds_t h = nullptr;
  int device = -1;
  yatt_rounds_t get() {
    int dev = 0;
    detail::cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
    if (h && dev != device) {
      yatt_rounds_destroy(h);
      h = nullptr;
    }
    if (!h) {
      detail::throw_status(yatt_rounds_create(&h));
      device = dev;
    }
    return h;
  }
  ~RoundsHandle() { yatt_rounds_destroy(h); }
};
thread_local RoundsHandle g_rounds;

ShardRoundReport shard_round_output(ShardState& state, int round, const RoundParams& params) {
  if (params.microbatch_size <= 0) throw ConfigError("microbatch_size must be positive");
  const std::int64_t n = static_cast<std::int64_t>(state.samples.size());
  yatt_rounds_t h = g_rounds.get();
  yatt_rounds_io io{};
  detail::throw_status(yatt_rounds_stage(h, n, 1, &io));
  for (std::int64_t i = 0; i < n; ++i) {
    const ShardSampleState& s = state.samples[static_cast<size_t>(i)];
    io.sample_id[i] = s.sample_id;
    io.prompt_len[i] = s.prompt_len_tokens;
    io.accepted[i] = s.accepted ? 1 : 0;
  }
  const yatt_round_params p = to_c(params);
  const std::int64_t off[2] = {0, n};
  detail::throw_status(yatt_rounds_run(h, n, off, 1, state.controller_rank, state.step_index,
                                       round, 1, &p, 0, nullptr));
  yatt_rounds_view v{};
  detail::throw_status(yatt_rounds_result(h, &v));
  for (std::int64_t i = 0; i < n; ++i) {
    ShardSampleState& s = state.samples[static_cast<size_t>(i)];
    if (s.accepted) continue;  // untouched by the round
    s.out_len_tokens = io.out_len[i];
    s.accepted = io.accepted_out[i] != 0;
    s.accepted_round = io.accepted_round[i];
  }
  return from_c(v.reports[0], v.microbatches);
}

ShardState make_shard_state(const workload::RolloutBatch& batch, int num_controllers,
                            int controller_rank) {
  const workload::ShardRange range = workload::shard_dataset(
      static_cast<std::uint64_t>(batch.samples.size()), num_controllers, controller_rank);
  ShardState shard;
  shard.controller_rank = controller_rank;
  shard.step_index = batch.step_index;
  shard.samples.reserve(range.size());
  for (std::uint64_t i = range.begin; i < range.end; ++i) {
    const workload::RolloutSample& s = batch.samples[i];
    shard.samples.push_back(ShardSampleState{s.sample_id, s.prompt_len_tokens,
                                             s.target_out_len_tokens, s.accepted,
                                             s.accepted_round});
  }
  return shard;
}

RoundReduction reduce_round_reports(const std::vector<ShardRoundReport>& reports) {
  RoundReduction r;
  for (const ShardRoundReport& rep : reports) {
    r.active += rep.active_count;
    r.pending += rep.pending_count;
    r.forced_accepts += rep.forced_accept_count;
    r.train_units += rep.accepted_train_units;
    r.score_tokens += rep.accepted_score_tokens;
  }
  return r;
}

// Host threads for the pack / copy-back loops of a call: 1 below 8,192
// samples (the fork costs more than it saves), else 2 — measured on the B200
// box at configs[4] (16,384 samples): round loop 1 thread 0.095 ms, 2 0.080,
// 4 0.084, 8 0.088 (the batch sits in the calling core's cache; more threads
// mostly add cross-core traffic).  YATT_HOST_THREADS overrides.
static int host_threads(std::int64_t n) {
  static const int cap = [] {
    const char* e = std::getenv("YATT_HOST_THREADS");
    const int hw = int(std::thread::hardware_concurrency());
    return e ? std::max(1, std::atoi(e)) : std::max(1, std::min(2, hw));
  }();
  return n >= 8192 ? cap : 1;
}

// The round loop over host samples: smp[0..n) split into the controller
// shards `off` (all shards of one process), or, with a peer group, this
// rank's single shard with every rank's reports gathered once
// (yatt_peer_rounds_run).
static std::vector<std::vector<ShardRoundReport>> rounds_impl(
    workload::RolloutSample* smp, std::int64_t n, const std::vector<std::int64_t>& off,
    int num_controllers, int step_index, const RoundParams& params,
    std::vector<int>* first_round_lengths, yatt_peer_t peer) {
  yatt_rounds_t h = g_rounds.get();
  yatt_rounds_io io{};
  detail::throw_status(yatt_rounds_stage(h, n, num_controllers, &io));
  // AoS -> SoA into the pinned stage; large batches split over a few host
  // threads (the reference runs one host thread per shard, simcore.cpp:470)
  const int nt = host_threads(n);
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
  for (std::int64_t i = 0; i < n; ++i) {
    io.sample_id[i] = smp[i].sample_id;
    io.prompt_len[i] = smp[i].prompt_len_tokens;
    io.accepted[i] = smp[i].accepted ? 1 : 0;
  }
  const yatt_round_params p = to_c(params);
  if (peer == nullptr)
    detail::throw_status(yatt_rounds_run(h, n, off.data(), num_controllers, 0, step_index, 1, 0,
                                         &p, first_round_lengths ? 1 : 0, nullptr));
  else
    detail::throw_status(
        yatt_peer_rounds_run(peer, h, n, step_index, &p, first_round_lengths ? 1 : 0, nullptr));
  yatt_rounds_view v{};
  detail::throw_status(yatt_rounds_result(h, &v));
  std::vector<std::vector<ShardRoundReport>> all(static_cast<size_t>(v.rounds));
  const yatt_mb_agg* mb = v.microbatches;
  const int shards = v.num_shards;  // == num_controllers, or the world with a peer group
  for (int r = 0; r < v.rounds; ++r) {
    auto& reports = all[static_cast<size_t>(r)];
    reports.reserve(static_cast<size_t>(shards));
    for (int s = 0; s < shards; ++s) {
      const yatt_round_report& rep = v.reports[static_cast<size_t>(r) * shards + s];
      reports.push_back(from_c(rep, mb));
      mb += rep.num_microbatches;
    }
  }
  if (first_round_lengths) first_round_lengths->resize(static_cast<size_t>(n));
#pragma omp parallel for num_threads(nt) schedule(static) if (nt > 1)
  for (std::int64_t i = 0; i < n; ++i) {  // copy_back (simcore.cpp:107-119)
    if (smp[i].accepted) {  // accepted before the step: untouched
      if (first_round_lengths) (*first_round_lengths)[static_cast<size_t>(i)] = smp[i].target_out_len_tokens;
      continue;
    }
    smp[i].target_out_len_tokens = io.out_len[i];
    smp[i].accepted = io.accepted_out[i] != 0;
    smp[i].accepted_round = io.accepted_round[i];
    if (first_round_lengths) (*first_round_lengths)[static_cast<size_t>(i)] = io.first_round_len[i];
  }
  return all;
}


std::vector<std::vector<ShardRoundReport>> run_rollout_rounds(workload::RolloutBatch& batch,
                                                              int num_controllers,
                                                              const RoundParams& params,
                                                              std::vector<int>* first_round_lengths) {
  params.out_dist.validate();
  if (params.max_rounds < 1) throw ConfigError("max_rounds must be at least 1");
  if (num_controllers < 1) throw ConfigError("num_controllers must be positive");
  if (params.microbatch_size <= 0) throw ConfigError("microbatch_size must be positive");
  const std::int64_t n = static_cast<std::int64_t>(batch.samples.size());
  std::vector<std::int64_t> off(static_cast<size_t>(num_controllers) + 1, 0);
  for (int r = 0; r < num_controllers; ++r) {
    const workload::ShardRange sr =
        workload::shard_dataset(static_cast<std::uint64_t>(n), num_controllers, r);
    off[static_cast<size_t>(r)] = static_cast<std::int64_t>(sr.begin);
    off[static_cast<size_t>(r) + 1] = static_cast<std::int64_t>(sr.end);
  }
  return rounds_impl(batch.samples.data(), n, off, num_controllers, batch.step_index, params,
                     first_round_lengths, nullptr);
}

}  // namespace sim

// ------------------------------------------------------------ balancer ----
namespace balancer {

double simulated_workload(double len_tokens) { return len_tokens * len_tokens; }

BatchingPlan sort_and_bucket(const std::vector<int>& lengths, int batch_size, std::uint64_t seed) {
  if (batch_size <= 0) throw ConfigError("batch_size must be positive");
  const std::int64_t n = static_cast<std::int64_t>(lengths.size());
  const std::int64_t nb = (n + batch_size - 1) / batch_size;
  std::vector<std::uint32_t> flat(static_cast<size_t>(n));
  std::vector<std::int64_t> off(static_cast<size_t>(nb) + 1);
  detail::throw_status(yatt_sort_and_bucket_host(lengths.data(), n, batch_size, seed, flat.data(),
                                                 off.data()));
  BatchingPlan plan;
  plan.batch_size = batch_size;
  plan.shuffle_seed = seed;
  plan.buckets.reserve(static_cast<size_t>(nb));
  for (std::int64_t b = 0; b < nb; ++b)
    plan.buckets.emplace_back(flat.begin() + off[static_cast<size_t>(b)],
                              flat.begin() + off[static_cast<size_t>(b) + 1]);
  return plan;
}

double padding_waste(const BatchingPlan& plan, const std::vector<int>& lengths) {
  double real = 0, padded = 0;
  for (const auto& bucket : plan.buckets) {
    int longest = 0;
    for (std::uint32_t i : bucket) {
      longest = std::max(longest, lengths.at(i));
      real += simulated_workload(lengths.at(i));
    }
    padded += static_cast<double>(bucket.size()) * simulated_workload(longest);
  }
  return padded == 0 ? 0.0 : 1.0 - real / padded;
}

double waste_bound(int batch_size) {
  if (batch_size <= 0) throw ConfigError("batch_size must be positive");
  const double keep = static_cast<double>(batch_size - 1) / batch_size;
  return 1.0 - keep * keep;
}

double distribution_bias_check(const BatchingPlan& plan, const std::vector<int>& lengths,
                               int window_buckets) {
  if (window_buckets <= 0) throw ConfigError("window_buckets must be positive");
  if (plan.buckets.empty() || lengths.empty()) return 0;
  const double n = static_cast<double>(lengths.size());
  double sum = 0;
  for (int l : lengths) sum += l;
  const double mu = sum / n;
  double var = 0;
  for (int l : lengths) var += (l - mu) * (l - mu);
  const double sd = std::sqrt(var / n);
  if (sd == 0) return 0;
  const int nb = static_cast<int>(plan.buckets.size());
  const int w = std::min(window_buckets, nb);
  double worst = 0;
  for (int s = 0; s + w <= nb; ++s) {
    double ws = 0;
    size_t cnt = 0;
    for (int b = s; b < s + w; ++b)
      for (std::uint32_t i : plan.buckets[static_cast<size_t>(b)]) {
        ws += lengths.at(i);
        ++cnt;
      }
    if (cnt) worst = std::max(worst, std::abs(ws / static_cast<double>(cnt) - mu) / sd);
  }
  return worst;
}

}  // namespace balancer

// ---------------------------------------------------------- experience ----
namespace experience {

void token_logprob_stats(const std::uint16_t* pol, const std::uint16_t* ref,
                         const std::int32_t* tgt, const std::uint8_t* mask, std::int64_t rows,
                         int vocab, KlEstimator kl, const TokenStats& out, void* stream) {
  detail::throw_status(yatt_token_stats(pol, ref, tgt, mask, rows, vocab, static_cast<int>(kl),
                                        out.logp, out.ref_logp, out.entropy, out.kl, stream));
}

void GrpoConfig::validate() const {
  if (group_size <= 0) throw ConfigError("group_size must be positive");
  if (!(eps >= 0)) throw ConfigError("eps must be non-negative");
}

void grpo_advantages(const float* rewards, std::int64_t n, std::uint64_t first_id,
                     const GrpoConfig& c, float* adv, const double* moments, void* stream) {
  c.validate();
  detail::throw_status(yatt_grpo_advantages(rewards, n, first_id, c.group_size, c.eps,
                                            c.norm_by_std ? 1 : 0, moments, adv, stream));
}

void GaeConfig::validate() const {
  if (!(gamma >= 0) || !(lam >= 0)) throw ConfigError("gamma and lam must be non-negative");
}

std::size_t gae_workspace_bytes(std::int64_t n_tokens) { return yatt_gae_workspace_bytes(n_tokens); }

void gae(const float* values, const float* rewards, const std::uint8_t* mask,
         const std::int64_t* cu, std::int64_t n_seqs, std::int64_t n_tokens, const GaeConfig& c,
         float* adv, float* ret, void* ws, std::size_t ws_bytes, void* stream,
         double* moments) {
  c.validate();
  if (moments)
    detail::throw_status(yatt_gae_with_moments(values, rewards, mask, cu, n_seqs, n_tokens,
                                               c.gamma, c.lam, adv, ret, moments, ws, ws_bytes,
                                               stream));
  else
    detail::throw_status(yatt_gae(values, rewards, mask, cu, n_seqs, n_tokens, c.gamma, c.lam,
                                  adv, ret, ws, ws_bytes, stream));
}

void PolicyLossConfig::validate() const {
  if (!(clip_low >= 0 && clip_low < 1)) throw ConfigError("clip_low must lie in [0, 1)");
  if (!(clip_high >= 0)) throw ConfigError("clip_high must be non-negative");
  if (clip_ratio_c != 0 && !(clip_ratio_c > 1)) throw ConfigError("clip_ratio_c must be > 1 or 0");
}

namespace {
yatt_loss_config to_c(const PolicyLossConfig& c) {
  return yatt_loss_config{c.clip_low, c.clip_high, c.clip_ratio_c, c.kl_coef, c.entropy_coef,
                          static_cast<std::int32_t>(c.aggregation)};
}
}  // namespace

std::size_t policy_loss_workspace_bytes() { return yatt_policy_loss_workspace_bytes(0, 0, 0); }

void policy_loss(const float* logp, const float* old_logp, const float* adv, const float* kl,
                 const float* ent, const std::uint8_t* mask, std::int64_t n,
                 const std::int64_t* cu, std::int64_t nseq, const PolicyLossConfig& c,
                 LossSums* sums, void* ws, std::size_t ws_bytes, void* stream) {
  static_assert(sizeof(LossSums) == sizeof(yatt_loss_sums), "LossSums layout");
  c.validate();
  const yatt_loss_config cc = to_c(c);
  detail::throw_status(yatt_policy_loss(logp, old_logp, adv, kl, ent, mask, n, cu, nseq, &cc,
                                        reinterpret_cast<yatt_loss_sums*>(sums), ws, ws_bytes,
                                        stream));
}

double finalize_loss(const LossSums& s, const PolicyLossConfig& c) {
  const yatt_loss_config cc = to_c(c);
  return yatt_loss_finalize(reinterpret_cast<const yatt_loss_sums*>(&s), &cc);
}

void policy_logits_grad(const std::uint16_t* pol, const std::uint16_t* ref,
                        const std::int32_t* tgt, const TokenStats& st, const float* old_logp,
                        const float* adv, const std::uint8_t* mask, std::int64_t rows, int vocab,
                        const std::int64_t* cu, std::int64_t nseq, const PolicyLossConfig& c,
                        KlEstimator kl, double norm, float* coef, std::uint16_t* grad,
                        void* stream) {
  c.validate();
  const yatt_loss_config cc = to_c(c);
  const int mode = static_cast<int>(kl);
  detail::throw_status(yatt_policy_grad_coef(pol, ref, tgt, st.logp, st.ref_logp, old_logp, adv,
                                             st.entropy, st.kl, mask, rows, vocab, cu, nseq, &cc,
                                             mode, norm, coef, stream));
  detail::throw_status(yatt_logits_backward(pol, kl == KlEstimator::kFull ? ref : nullptr, tgt,
                                            mask, rows, vocab, coef,
                                            kl == KlEstimator::kFull ? 1 : 0, grad, stream));
}

std::size_t policy_loss_grad_workspace_bytes(std::int64_t rows, LossAggregation a) {
  return yatt_policy_loss_grad_workspace_bytes(rows, static_cast<int32_t>(a));
}

void policy_loss_grad(const std::uint16_t* pol, const std::uint16_t* ref, const std::int32_t* tgt,
                      const std::uint8_t* mask, const float* ref_logp, const float* old_logp, const float* adv,
                      std::int64_t rows, int vocab, const std::int64_t* cu, std::int64_t nseq,
                      const PolicyLossConfig& c, KlEstimator kl, double norm,
                      const TokenStats& out, std::uint16_t* grad, void* ws, std::size_t ws_bytes,
                      void* stream) {
  c.validate();
  const yatt_loss_config cc = to_c(c);
  detail::throw_status(yatt_policy_loss_grad(pol, ref, tgt, mask, ref_logp, old_logp, adv, rows, vocab,
                                             cu, nseq, &cc, static_cast<int>(kl), norm, out.logp,
                                             out.entropy, out.kl, grad, ws, ws_bytes, stream));
}

std::size_t lmhead_workspace_bytes(std::int64_t rows, int vocab, int n_split) {
  return yatt_lmhead_workspace_bytes(rows, vocab, n_split);
}

void lmhead_token_stats(const std::uint16_t* hidden, const std::uint16_t* w,
                        const std::int32_t* tgt, std::int64_t rows, int d, int vocab, int n_split,
                        float* logp, float* ent, float* lse, void* ws, std::size_t ws_bytes,
                        void* stream) {
  detail::throw_status(yatt_lmhead_token_stats(hidden, w, tgt, rows, d, vocab, n_split, logp, ent,
                                               lse, ws, ws_bytes, stream));
}

void gather_payload(const std::vector<PayloadArray>& arrays, const std::int64_t* old_cu,
                    const CompactionBuffers& plan, std::int64_t max_kept,
                    const std::int64_t* dst_offset, void* stream) {
  if (arrays.empty()) return;
  std::vector<const void*> src;
  std::vector<void*> dst;
  std::vector<std::int32_t> esz;
  for (const auto& a : arrays) {
    src.push_back(a.src);
    dst.push_back(a.dst);
    esz.push_back(a.elem_bytes);
  }
  // counts[0] = kept samples (device), the gather's loop bound
  detail::throw_status(yatt_gather_varlen_multi(static_cast<std::int32_t>(arrays.size()),
                                                src.data(), dst.data(), esz.data(), old_cu,
                                                plan.index_map, plan.new_cu, plan.counts, max_kept,
                                                dst_offset, stream));
}

PeerGroup::PeerGroup(int world, int rank)
    : handle_(YATT_PEER_HANDLE_BYTES), world_(world), rank_(rank) {
  yatt_peer_t p = nullptr;
  detail::throw_status(yatt_peer_create(world, rank, &p, handle_.data()));
  h_ = p;
}

PeerGroup::~PeerGroup() { yatt_peer_destroy(static_cast<yatt_peer_t>(h_)); }

void PeerGroup::connect(const std::vector<std::uint8_t>& all) {
  detail::throw_status(yatt_peer_connect(static_cast<yatt_peer_t>(h_), all.data()));
}

void PeerGroup::allreduce(const double* in, int n, double* out, void* stream) {
  detail::throw_status(yatt_peer_allreduce_f64(static_cast<yatt_peer_t>(h_), in, n, out, stream));
}

void PeerGroup::scan(const std::int64_t* in, int n, std::int64_t* prefix, std::int64_t* total,
                     void* stream) {
  detail::throw_status(
      yatt_peer_scan_i64(static_cast<yatt_peer_t>(h_), in, n, prefix, total, stream));
}

void PeerGroup::allgather(const std::int64_t* in, int n, std::int64_t* out, void* stream) {
  detail::throw_status(
      yatt_peer_allgather_i64(static_cast<yatt_peer_t>(h_), in, n, out, stream));
}

void PeerGroup::policy_loss(const float* logp, const float* old_logp, const float* adv,
                            const float* kl, const float* ent, const std::uint8_t* mask,
                            std::int64_t n, const std::int64_t* cu, std::int64_t nseq,
                            const PolicyLossConfig& c, LossSums* sums, void* ws,
                            std::size_t ws_bytes, void* stream) {
  c.validate();
  const yatt_loss_config cc = to_c(c);
  detail::throw_status(yatt_policy_loss_allreduce(
      static_cast<yatt_peer_t>(h_), logp, old_logp, adv, kl, ent, mask, n, cu, nseq, &cc,
      reinterpret_cast<yatt_loss_sums*>(sums), ws, ws_bytes, stream));
}

std::size_t PeerGroup::straddle_workspace_bytes(std::int64_t n, std::uint64_t first_id,
                                                int G) const {
  return yatt_straddle_workspace_bytes(n, first_id, G, world_);
}

void PeerGroup::grpo_advantages(const float* rewards, std::int64_t n, std::uint64_t first_id,
                                const GrpoConfig& c, float* adv, void* ws, std::size_t ws_bytes,
                                void* stream) {
  c.validate();
  detail::throw_status(yatt_peer_grpo_advantages(static_cast<yatt_peer_t>(h_), rewards, n,
                                                 first_id, c.group_size, c.eps,
                                                 c.norm_by_std ? 1 : 0, adv, ws, ws_bytes,
                                                 stream));
}

void PeerGroup::dynamic_sampling_filter(const float* rewards, const std::int64_t* lens,
                                        std::int64_t n, std::uint64_t first_id, int G,
                                        const CompactionBuffers& o, void* ws,
                                        std::size_t ws_bytes, void* stream) {
  detail::throw_status(yatt_peer_filter_compact(static_cast<yatt_peer_t>(h_), rewards, lens, n,
                                                first_id, G, o.keep_groups, o.index_map,
                                                o.new_cu, o.counts, ws, ws_bytes, stream));
}

std::vector<std::vector<sim::ShardRoundReport>> PeerGroup::run_rollout_rounds(
    std::vector<workload::RolloutSample>& shard_samples, int step_index,
    const sim::RoundParams& params, std::vector<int>* first_round_lengths) {
  params.out_dist.validate();
  if (params.max_rounds < 1) throw ConfigError("max_rounds must be at least 1");
  if (params.microbatch_size <= 0) throw ConfigError("microbatch_size must be positive");
  const std::int64_t n = static_cast<std::int64_t>(shard_samples.size());
  return sim::rounds_impl(shard_samples.data(), n, {0, n}, 1, step_index, params,
                          first_round_lengths, static_cast<yatt_peer_t>(h_));
}

int PeerGroup::status() const {
  std::int32_t s = 0;
  detail::throw_status(yatt_peer_status(static_cast<yatt_peer_t>(h_), &s));
  return s;
}

std::size_t dynamic_sampling_workspace_bytes(std::int64_t n) {
  return yatt_filter_compact_workspace_bytes(n);
}

void dynamic_sampling_filter(const float* rewards, const std::int64_t* lens, std::int64_t n,
                             int G, const CompactionBuffers& o, void* ws, std::size_t ws_bytes,
                             void* stream) {
  detail::throw_status(yatt_filter_compact(rewards, lens, n, G, o.keep_groups, o.index_map,
                                           o.new_cu, o.counts, ws, ws_bytes, stream));
}

void dynamic_sampling_boundary_record(const float* rewards, std::int64_t n,
                                      std::uint64_t first_id, int G, std::int64_t* record,
                                      void* stream) {
  detail::throw_status(yatt_filter_boundary_record(rewards, n, first_id, G, record, stream));
}

void dynamic_sampling_filter_sharded(const float* rewards, const std::int64_t* lens,
                                     std::int64_t n, std::uint64_t first_id, int G,
                                     const std::int64_t* all_records, int world,
                                     const CompactionBuffers& o, void* ws, std::size_t ws_bytes,
                                     void* stream) {
  detail::throw_status(yatt_filter_compact_sharded(rewards, lens, n, first_id, G, all_records,
                                                   world, o.keep_groups, o.index_map, o.new_cu,
                                                   o.counts, ws, ws_bytes, stream));
}

std::int64_t grpo_num_local_groups(std::int64_t n, std::uint64_t first_id, int G) {
  if (G <= 0) throw ConfigError("group_size must be positive");
  return yatt_grpo_num_local_groups(n, first_id, G);
}

void grpo_group_moments(const float* rewards, std::int64_t n, std::uint64_t first_id, int G,
                        double* moments, void* stream) {
  detail::throw_status(yatt_grpo_group_moments(rewards, n, first_id, G, moments, stream));
}

void grpo_boundary_record(const double* moments, std::int64_t n, std::uint64_t first_id, int G,
                          double* record, void* stream) {
  detail::throw_status(yatt_grpo_boundary_record(moments, n, first_id, G, record, stream));
}

void grpo_merge_boundaries(double* moments, std::int64_t n, std::uint64_t first_id, int G,
                           const double* all_records, int world, void* stream) {
  detail::throw_status(
      yatt_grpo_merge_boundaries(moments, n, first_id, G, all_records, world, stream));
}

}  // namespace experience
}  // namespace yatt
