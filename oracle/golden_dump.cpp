// golden_dump.cpp — TEST INFRASTRUCTURE: golden vectors from the reference.
//
// Linked against oracle/_ref/libyatt_ref.a (the reference's own sources,
// compiled in place by oracle/Makefile).  Calls the reference functions on the
// path and writes their outputs to tests/golden/*.json; the C oracle and the
// B200 library are both checked bit-exactly against these files.
//   lengths.json     workload::sample_length_keyed, all four kinds
//   rejection.json   workload::rejection_process
//   shard.json       workload::shard_dataset (incl. error codes)
//   rollout_*.json   make_shard_state + shard_round_output rounds until no
//                    sample is pending (the loop of run_rlhf_step,
//                    simcore.cpp:470-484), every report + final sample state
//   buckets.json     balancer::sort_and_bucket + padding_waste
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "yatt/balancer.hpp"
#include "yatt/errors.hpp"
#include "yatt/simcore.hpp"
#include "yatt/workload.hpp"

using namespace yatt;

namespace {

template <typename T>
std::string arr(const std::vector<T>& v) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
  o << "]";
  return o.str();
}

std::string dbl(double d) {
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", d);
  return b;
}

void write(const std::string& path, const std::string& body) {
  std::ofstream f(path);
  f << body << "\n";
}

const char* kind_name(workload::DistKind k) {
  return k == workload::DistKind::kConstant  ? "constant"
         : k == workload::DistKind::kUniform ? "uniform"
         : k == workload::DistKind::kNormal  ? "normal"
                                             : "lognormal";
}

std::string dist_json(const workload::LengthDistribution& d) {
  std::ostringstream o;
  o << "{\"kind\":" << int(d.kind) << ",\"p1\":" << dbl(d.p1) << ",\"p2\":" << dbl(d.p2)
    << ",\"max_len\":" << d.max_len_tokens << "}";
  return o.str();
}

void dump_lengths(const std::string& dir) {
  using workload::DistKind;
  const std::vector<workload::LengthDistribution> dists = {
      {DistKind::kConstant, 480, 0, 1024},   {DistKind::kUniform, 1, 16384, 16384},
      {DistKind::kUniform, 1, 8192, 8192},   {DistKind::kNormal, 480, 120, 1024},
      {DistKind::kLogNormal, 5.0, 0.5, 4096}};
  std::ostringstream o;
  o << "{\"seed\":20250814,\"stream\":2,\"step\":3,\"round\":2,\"n\":4096,\"cases\":[";
  for (size_t k = 0; k < dists.size(); ++k) {
    std::vector<int> out;
    for (std::uint64_t id = 0; id < 4096; ++id)
      out.push_back(workload::sample_length_keyed(dists[k], 20250814, 2, 3, 2, id));
    o << (k ? "," : "") << "{\"dist\":" << dist_json(dists[k]) << ",\"name\":\""
      << kind_name(dists[k].kind) << "\",\"lengths\":" << arr(out) << "}";
  }
  o << "]}";
  write(dir + "/lengths.json", o.str());
}

void dump_rejection(const std::string& dir) {
  workload::RolloutBatch batch;
  batch.step_index = 5;
  std::vector<int> acc;
  for (int i = 0; i < 4096; ++i) {
    workload::RolloutSample s;
    s.sample_id = std::uint64_t(i) + 1000;
    s.accepted = (i % 7) == 3;
    acc.push_back(s.accepted);
    batch.samples.push_back(s);
  }
  std::ostringstream o;
  o << "{\"step\":5,\"id0\":1000,\"accepted\":" << arr(acc) << ",\"cases\":[";
  const std::vector<workload::RejectionConfig> cfgs = {{0.3, true, 16}, {0.4, false, 1},
                                                       {0.5, true, 8}, {0.0, false, 1}};
  bool first = true;
  for (const auto& c : cfgs)
    for (int round : {1, 2, 7}) {
      const auto flags = workload::rejection_process(batch, round, c, 20250814);
      std::vector<int> f(flags.begin(), flags.end());
      o << (first ? "" : ",") << "{\"rate\":" << dbl(c.reject_rate)
        << ",\"per_group\":" << c.per_group << ",\"group_size\":" << c.group_size
        << ",\"round\":" << round << ",\"flags\":" << arr(f) << "}";
      first = false;
    }
  o << "]}";
  write(dir + "/rejection.json", o.str());
}

void dump_shard(const std::string& dir) {
  std::ostringstream o;
  o << "{\"cases\":[";
  bool first = true;
  for (std::uint64_t total : {0ull, 1ull, 10ull, 128ull, 1037ull, 2048ull, 16384ull})
    for (int p : {0, 1, 2, 3, 4, 7, 8})
      for (int r : {-1, 0, 1, 2, 3, 6, 7, 8}) {
        int code = 0;
        std::uint64_t b = 0, e = 0;
        try {
          const auto s = workload::shard_dataset(total, p, r);
          b = s.begin;
          e = s.end;
        } catch (const RankOutOfRange&) {
          code = 2;
        } catch (const ConfigError&) {
          code = 1;
        }
        o << (first ? "" : ",") << "[" << total << "," << p << "," << r << "," << code << ","
          << b << "," << e << "]";
        first = false;
      }
  o << "]}";
  write(dir + "/shard.json", o.str());
}

struct RolloutCase {
  std::string name;
  int n;
  int step;
  workload::LengthDistribution prompt, out;
  workload::RejectionConfig rej;
  std::uint64_t seed;
  int mb, max_rounds;
  std::vector<int> controllers;
};

void dump_rollout(const std::string& dir, const RolloutCase& c) {
  std::ostringstream o;
  o << "{\"name\":\"" << c.name << "\",\"n\":" << c.n << ",\"step\":" << c.step
    << ",\"prompt_dist\":" << dist_json(c.prompt) << ",\"out_dist\":" << dist_json(c.out)
    << ",\"reject_rate\":" << dbl(c.rej.reject_rate) << ",\"per_group\":" << c.rej.per_group
    << ",\"group_size\":" << c.rej.group_size << ",\"seed\":" << c.seed << ",\"mb\":" << c.mb
    << ",\"max_rounds\":" << c.max_rounds << ",\"runs\":[";
  for (size_t ci = 0; ci < c.controllers.size(); ++ci) {
    const int P = c.controllers[ci];
    workload::RolloutBatch batch;
    batch.step_index = c.step;
    for (int i = 0; i < c.n; ++i) {
      workload::RolloutSample s;
      s.sample_id = std::uint64_t(c.step) * std::uint64_t(c.n) + std::uint64_t(i);
      s.prompt_len_tokens = workload::sample_length_keyed(c.prompt, c.seed, workload::kPromptLenStream,
                                                          std::uint64_t(c.step), 0, s.sample_id);
      batch.samples.push_back(s);
    }
    std::vector<sim::ShardState> shards;
    for (int r = 0; r < P; ++r) shards.push_back(sim::make_shard_state(batch, P, r));
    const sim::RoundParams params{c.out, c.rej, c.seed, c.mb, c.max_rounds};
    o << (ci ? "," : "") << "{\"controllers\":" << P << ",\"prompt_len\":[";
    for (int i = 0; i < c.n; ++i) o << (i ? "," : "") << batch.samples[size_t(i)].prompt_len_tokens;
    o << "],\"rounds\":[";
    for (int round = 1;; ++round) {
      long long pending = 0;
      o << (round > 1 ? "," : "") << "[";
      for (int r = 0; r < P; ++r) {
        const sim::ShardRoundReport rep = sim::shard_round_output(shards[size_t(r)], round, params);
        pending += rep.pending_count;
        std::vector<long long> mbs;
        for (const auto& m : rep.microbatches) {
          mbs.push_back(m.controller_rank);
          mbs.push_back(m.mb_index);
          mbs.push_back(m.sample_count);
          mbs.push_back(m.max_out_len_tokens);
          mbs.push_back(m.score_tokens);
        }
        o << (r ? "," : "") << "{\"report\":[" << rep.controller_rank << "," << rep.round << ","
          << rep.active_count << "," << rep.newly_accepted_count << ","
          << rep.forced_accept_count << "," << rep.pending_count << ","
          << rep.accepted_score_tokens << "," << rep.accepted_train_units
          << "],\"mbs\":" << arr(mbs) << "}";
      }
      o << "]";
      if (pending == 0) break;
    }
    std::vector<int> out_len, acc, acc_round;
    for (const auto& sh : shards)
      for (const auto& s : sh.samples) {
        out_len.push_back(s.out_len_tokens);
        acc.push_back(s.accepted);
        acc_round.push_back(s.accepted_round);
      }
    o << "],\"final_out_len\":" << arr(out_len) << ",\"final_accepted\":" << arr(acc)
      << ",\"final_accepted_round\":" << arr(acc_round) << "}";
  }
  o << "]}";
  write(dir + "/rollout_" + c.name + ".json", o.str());
}

void dump_buckets(const std::string& dir) {
  std::ostringstream o;
  o << "{\"cases\":[";
  bool first = true;
  for (int n : {0, 1, 11, 64, 1000, 4096, 16384})
    for (int B : {1, 4, 16})
      for (std::uint64_t seed : {3ull, 20250814ull}) {
        std::vector<int> lengths(static_cast<size_t>(n));
        std::mt19937_64 rng(seed + std::uint64_t(n));
        for (auto& l : lengths) l = 1 + int(rng() % (n > 1000 ? 16384 : 64));  // many ties
        const balancer::BatchingPlan plan = balancer::sort_and_bucket(lengths, B, seed);
        std::vector<std::uint32_t> flat;
        std::vector<long long> off{0};
        for (const auto& b : plan.buckets) {
          flat.insert(flat.end(), b.begin(), b.end());
          off.push_back(static_cast<long long>(flat.size()));
        }
        o << (first ? "" : ",") << "{\"n\":" << n << ",\"B\":" << B << ",\"seed\":" << seed
          << ",\"lengths\":" << arr(lengths) << ",\"flat\":" << arr(flat)
          << ",\"offsets\":" << arr(off)
          << ",\"waste\":" << dbl(balancer::padding_waste(plan, lengths)) << "}";
        first = false;
      }
  o << "]}";
  write(dir + "/buckets.json", o.str());
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  using workload::DistKind;
  dump_lengths(dir);
  dump_rejection(dir);
  dump_shard(dir);
  // BASELINE configs[0]: 16 prompts x 8 responses (GRPO group filter G=8).
  dump_rollout(dir, {"config1", 128, 0, {DistKind::kUniform, 16, 64, 4096},
                     {DistKind::kUniform, 1, 256, 256}, {0.3, true, 8}, 20250814, 8, 4,
                     {1, 2, 4, 8}});
  // configs[4]: 1024 prompts x 16 responses, T=16k, prompt 64.
  dump_rollout(dir, {"config5", 16384, 1, {DistKind::kConstant, 64, 0, 64},
                     {DistKind::kUniform, 1, 16384, 16384}, {0.3, true, 16}, 20250814, 16, 4,
                     {1, 8}});
  dump_rollout(dir, {"normal", 2048, 2, {DistKind::kUniform, 32, 512, 4096},
                     {DistKind::kNormal, 2048, 512, 4096}, {0.25, false, 1}, 7, 8, 64, {4}});
  dump_rollout(dir, {"lognormal_p3", 96, 3, {DistKind::kConstant, 40, 0, 40},
                     {DistKind::kLogNormal, 5.0, 0.5, 4096}, {0.5, true, 4}, 11, 5, 3, {3}});
  dump_buckets(dir);
  std::printf("golden vectors written to %s\n", dir.c_str());
  return 0;
}
