// small_call_latency.cpp — per-call latency of sim::run_rollout_rounds (the
// drop-in's round loop) at the small batch sizes the reference's scenario
// tests use, with the C-ABI phases split out (stage / run / result).
// Build: g++ -std=c++20 -O2 -I include tools/small_call_latency.cpp \
//        -L paper_2508_07970_b200 -lyatt_b200 -Wl,-rpath,$PWD/paper_2508_07970_b200
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "yatt/simcore.hpp"
#include "yatt/workload.hpp"
#include "yatt_cuda.h"

using namespace yatt;
using clk = std::chrono::steady_clock;

int main() {
  for (int n : {8, 64, 512, 4096}) {
    for (int P : {1, 4}) {
      sim::RoundParams params;
      params.out_dist = {workload::DistKind::kUniform, 1, 4096, 4096};
      params.rejection = {0.3, true, 8};
      params.seed = 7;
      params.microbatch_size = 4;
      params.max_rounds = 4;
      auto make = [&] {
        workload::RolloutBatch b;
        b.step_index = 3;
        for (int i = 0; i < n; ++i) {
          workload::RolloutSample s;
          s.sample_id = std::uint64_t(i);
          s.prompt_len_tokens = 32;
          b.samples.push_back(s);
        }
        return b;
      };
      for (int w = 0; w < 20; ++w) {
        auto b = make();
        sim::run_rollout_rounds(b, P, params);
      }
      std::vector<double> t;
      for (int it = 0; it < 400; ++it) {
        auto b = make();
        const auto t0 = clk::now();
        sim::run_rollout_rounds(b, P, params);
        t.push_back(std::chrono::duration<double, std::micro>(clk::now() - t0).count());
      }
      std::sort(t.begin(), t.end());
      std::printf("{\"n\": %d, \"P\": %d, \"p50_us\": %.1f, \"p10_us\": %.1f, \"p90_us\": %.1f}\n", n,
                  P, t[t.size() / 2], t[t.size() / 10], t[t.size() * 9 / 10]);
    }
  }
  return 0;
}
