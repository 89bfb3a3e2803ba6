// ref_timing.cpp — TEST/BASELINE INFRASTRUCTURE (SURVEY.md §8d "CPU path
// timed beside it", item (i)): times the reference's own integer path,
// compiled from its sources (oracle/_ref/libyatt_ref.a), on configs[4]'s
// dynamic-sampling batch (1,024 prompts x 16 responses, 64-token prompts,
// responses U[1, 16384], per-group rejection 0.3, microbatches of 16):
//   * the round loop of run_rlhf_step (simcore.cpp:470-491): shard_round_output
//     for P controller shards, one host thread per shard (P threads), until no
//     shard has pending samples (max_rounds 4 forces acceptance);
//   * rejection_process (workload.cpp:145-167) over the batch, one thread;
//   * sort_and_bucket (balancer.cpp:16-41) of the accepted lengths, B = 16.
// Timing: the median of 5 runs of >= 0.5 s each, per operation.
// Usage: ref_timing [P]   -> one JSON line.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
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

int main(int argc, char** argv) {
  const int P = argc > 1 ? std::atoi(argv[1]) : 8;
  const int prompts = 1024, G = 16, n = prompts * G;
  const std::uint64_t seed = 20250814;
  workload::RolloutBatch batch;
  batch.step_index = 1;
  for (int i = 0; i < n; ++i) {
    workload::RolloutSample s;
    s.sample_id = std::uint64_t(n) + std::uint64_t(i);
    s.prompt_len_tokens = 64;
    batch.samples.push_back(s);
  }
  sim::RoundParams params;
  params.out_dist.kind = workload::DistKind::kUniform;
  params.out_dist.p1 = 1;
  params.out_dist.p2 = 16384;
  params.out_dist.max_len_tokens = 16384;
  params.rejection.reject_rate = 0.3;
  params.rejection.per_group = true;
  params.rejection.group_size = G;
  params.seed = seed;
  params.microbatch_size = 16;
  params.max_rounds = 4;

  // shard round loop, P threads: fresh shard states per operation
  int rounds = 0;
  long long units = 0;
  auto mk_shards = [&] {
    std::vector<sim::ShardState> shards;
    for (int r = 0; r < P; ++r) shards.push_back(sim::make_shard_state(batch, P, r));
    return shards;
  };
  double first_ms = 0.0;
  const double loop_ms = median_ms(mk_shards, [&](std::vector<sim::ShardState>& shards) {
    std::vector<sim::ShardRoundReport> reports(static_cast<size_t>(P));
    int round = 1;
    long long u = 0;
    while (true) {
      const auto tr = clk::now();
      std::vector<std::thread> th;
      for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] { reports[size_t(r)] = sim::shard_round_output(shards[size_t(r)], round, params); });
      for (auto& t : th) t.join();
      if (round == 1) first_ms = ms_since(tr);
      int pending = 0;
      for (const auto& rep_ : reports) {
        pending += rep_.pending_count;
        u += rep_.accepted_train_units;
      }
      if (pending == 0) break;
      ++round;
    }
    rounds = round;
    units = u;
  });

  // rejection_process over the batch (one thread)
  const double rej_ms = median_ms([] { return 0; }, [&](int&) {
    volatile size_t keep = workload::rejection_process(batch, 1, params.rejection, seed).size();
    (void)keep;
  });

  // sort_and_bucket of n lengths (one thread)
  std::vector<int> lengths(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i)
    lengths[size_t(i)] = 64 + workload::sample_length_keyed(params.out_dist, seed,
                                                            workload::kOutputLenStream, 1, 1,
                                                            batch.samples[size_t(i)].sample_id);
  bool empty = false;
  const double sort_ms = median_ms([] { return 0; }, [&](int&) {
    const auto plan = balancer::sort_and_bucket(lengths, 16, seed);
    empty = empty || plan.buckets.empty();
  });
  if (empty) return 1;
  std::printf("{\"kind\": \"reference\", \"threads\": %d, \"samples\": %d, \"rounds\": %d, "
              "\"train_units\": %lld, \"shard_round_loop_ms\": %.4f, \"first_round_ms\": %.4f, "
              "\"rejection_process_ms\": %.4f, \"sort_and_bucket_ms\": %.4f}\n",
              P, n, rounds, units, loop_ms, first_ms, rej_ms, sort_ms);
  return 0;
}
