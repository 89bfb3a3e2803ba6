// integer_timing.cpp — configs[4]'s integer path through the drop-in C++ API
// (include/yatt + libyatt_b200.so), the counterpart of oracle/ref_timing.cpp
// (the reference's own code, one host thread per shard): 16,384 samples,
// 8 controller shards, sim::run_rollout_rounds (every round of every shard in
// one persistent kernel: one H2D copy, one launch, one synchronize) and
// balancer::sort_and_bucket.  Median of 5 runs after a warm-up; one JSON line.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "yatt/balancer.hpp"
#include "yatt/simcore.hpp"
#include "yatt/workload.hpp"
#include "yatt_cuda.h"

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
  // Where a call's time goes (C ABI underneath sim::run_rollout_rounds),
  // single-threaded here (the API splits the pack / copy-back loops over 2
  // host threads): packing into the pinned stage, the device call (the
  // persistent kernel reads the stage in place, results in mapped host
  // memory, one synchronize), unpacking.
  double pack_ms = 0, call_ms = 0, unpack_ms = 0;
  {
    yatt_rounds_t h = nullptr;
    if (yatt_rounds_create(&h) != 0) return 1;
    std::vector<std::int64_t> off(P + 1);
    for (int r = 0; r <= P; ++r) off[r] = std::int64_t(n) * r / P;
    const yatt_round_params cp{{int32_t(params.out_dist.kind), params.out_dist.max_len_tokens,
                                params.out_dist.p1, params.out_dist.p2},
                               {params.rejection.reject_rate, 1, G}, seed, 16, 4};
    std::vector<double> a, b, c;
    for (int it = 0; it < 300; ++it) {
      auto batch = make_batch();
      const auto t0 = clk::now();
      yatt_rounds_io io{};
      yatt_rounds_stage(h, n, P, &io);
      for (int i = 0; i < n; ++i) {
        const auto& x = batch.samples[std::size_t(i)];
        io.sample_id[i] = x.sample_id;
        io.prompt_len[i] = x.prompt_len_tokens;
        io.accepted[i] = x.accepted ? 1 : 0;
      }
      const auto t1 = clk::now();
      if (yatt_rounds_run(h, n, off.data(), P, 0, batch.step_index, 1, 0, &cp, 0, nullptr) != 0)
        return 1;
      const auto t2 = clk::now();
      yatt_rounds_view v{};
      yatt_rounds_result(h, &v);
      std::vector<std::vector<sim::ShardRoundReport>> all(std::size_t(v.rounds));
      const yatt_mb_agg* mb = v.microbatches;
      for (int r = 0; r < v.rounds; ++r)
        for (int q = 0; q < P; ++q) {
          const auto& rep = v.reports[std::size_t(r) * P + q];
          sim::ShardRoundReport o;
          o.active_count = rep.active_count;
          for (std::int64_t k = 0; k < rep.num_microbatches; ++k)
            o.microbatches.push_back({mb[k].controller_rank, mb[k].mb_index, mb[k].sample_count,
                                      mb[k].max_out_len_tokens, mb[k].score_tokens});
          mb += rep.num_microbatches;
          all[std::size_t(r)].push_back(std::move(o));
        }
      for (int i = 0; i < n; ++i) {
        auto& x = batch.samples[std::size_t(i)];
        if (x.accepted) continue;
        x.target_out_len_tokens = io.out_len[i];
        x.accepted = io.accepted_out[i] != 0;
        x.accepted_round = io.accepted_round[i];
      }
      const auto t3 = clk::now();
      using ms = std::chrono::duration<double, std::milli>;
      a.push_back(ms(t1 - t0).count());
      b.push_back(ms(t2 - t1).count());
      c.push_back(ms(t3 - t2).count());
    }
    for (auto* v : {&a, &b, &c}) std::sort(v->begin(), v->end());
    pack_ms = a[a.size() / 2];
    call_ms = b[b.size() / 2];
    unpack_ms = c[c.size() / 2];
    yatt_rounds_destroy(h);
  }
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
              "\"sort_and_bucket_ms\": %.4f, \"round_loop_split_ms\": {\"pack\": %.4f, "
              "\"device_call\": %.4f, \"unpack\": %.4f}}\n",
              P, n, rounds, units, loop_ms, sort_ms, pack_ms, call_ms, unpack_ms);
  return 0;
}
