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

// BASELINE.md's timing method: the median of 5 runs, each repeating the
// operation until >= 0.5 s of timed work (per-op setup outside the timing);
// returns ms per operation.
template <class Setup, class Op>
static double median_ms(Setup setup, Op op) {
  std::vector<double> runs;
  for (int r = 0; r < 5; ++r) {
    double acc = 0.0;
    int k = 0;
    do {
      auto st = setup();
      const auto t0 = clk::now();
      op(st);
      acc += ms_since(t0);
      ++k;
    } while (acc < 500.0);
    runs.push_back(acc / k);
  }
  std::sort(runs.begin(), runs.end());
  return runs[2];
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
  int rounds = 0;
  long long units = 0;
  workload::RolloutBatch last;
  const double loop_ms = median_ms(make_batch, [&](workload::RolloutBatch& b) {
    const auto rr = sim::run_rollout_rounds(b, P, params);
    rounds = int(rr.size());
    units = 0;
    for (const auto& reps : rr)
      for (const auto& r : reps) units += r.accepted_train_units;
    last = b;
  });
  std::vector<int> lengths;
  for (const auto& s : last.samples) lengths.push_back(s.prompt_len_tokens + s.target_out_len_tokens);
  bool empty = false;
  const double sort_ms = median_ms([] { return 0; }, [&](int&) {
    const auto plan = balancer::sort_and_bucket(lengths, 16, seed);
    empty = empty || plan.buckets.empty();
  });
  if (empty) return 1;
  std::printf("{\"kind\": \"b200 (C++ drop-in API)\", \"shards\": %d, \"samples\": %d, "
              "\"rounds\": %d, \"train_units\": %lld, \"round_loop_ms\": %.4f, "
              "\"sort_and_bucket_ms\": %.4f}\n",
              P, n, rounds, units, loop_ms, sort_ms);
  return 0;
}
