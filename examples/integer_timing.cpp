// integer_timing.cpp — configs[4]'s integer path through the drop-in C++ API
// (include/yatt + libyatt_b200.so), the counterpart of oracle/ref_timing.cpp
// (the reference's own code, one host thread per shard): 16,384 samples,
// 8 controller shards, sim::run_rollout_rounds (every shard in one launch per
// round, state resident on the device, reports read back each round) and
// balancer::sort_and_bucket.  Best of 5 after a warm-up; one JSON line.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "yatt/balancer.hpp"
#include "yatt/simcore.hpp"
#include "yatt/workload.hpp"

using namespace yatt;
using clk = std::chrono::steady_clock;

static double ms_since(clk::time_point t0) {
  return std::chrono::duration<double, std::milli>(clk::now() - t0).count();
}

int main() {
  const int P = 8, G = 16, n = 1024 * G;
  const std::uint64_t seed = 20250814;
  auto make_batch = [&] {
    workload::RolloutBatch b;
    b.step_index = 1;
    for (int i = 0; i < n; ++i) {
      workload::RolloutSample s;
      s.sample_id = std::uint64_t(n) + std::uint64_t(i);
      s.prompt_len_tokens = 64;
      b.samples.push_back(s);
    }
    return b;
  };
  sim::RoundParams params;
  params.out_dist = {workload::DistKind::kUniform, 1, 16384, 16384};
  params.rejection = {0.3, true, G};
  params.seed = seed;
  params.microbatch_size = 16;
  params.max_rounds = 4;
  {
    auto warm = make_batch();
    sim::run_rollout_rounds(warm, P, params);
  }
  double best = 1e30;
  int rounds = 0;
  long long units = 0;
  workload::RolloutBatch last;
  for (int rep = 0; rep < 5; ++rep) {
    auto b = make_batch();
    const auto t0 = clk::now();
    const auto rr = sim::run_rollout_rounds(b, P, params);
    const double ms = ms_since(t0);
    if (ms < best) {
      best = ms;
      rounds = int(rr.size());
      units = 0;
      for (const auto& reps : rr)
        for (const auto& r : reps) units += r.accepted_train_units;
    }
    last = b;
  }
  std::vector<int> lengths;
  for (const auto& s : last.samples) lengths.push_back(s.prompt_len_tokens + s.target_out_len_tokens);
  balancer::sort_and_bucket(lengths, 16, seed);  // warm-up
  double best_sort = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    const auto t0 = clk::now();
    const auto plan = balancer::sort_and_bucket(lengths, 16, seed);
    best_sort = std::min(best_sort, ms_since(t0));
    if (plan.buckets.empty()) return 1;
  }
  std::printf("{\"kind\": \"b200 (C++ drop-in API)\", \"shards\": %d, \"samples\": %d, "
              "\"rounds\": %d, \"train_units\": %lld, \"round_loop_ms\": %.4f, "
              "\"sort_and_bucket_ms\": %.4f}\n",
              P, n, rounds, units, best, best_sort);
  return 0;
}
