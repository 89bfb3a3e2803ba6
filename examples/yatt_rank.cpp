// yatt_rank.cpp — one WeChat-YATT parallel-controller rank written against the
// drop-in C++ API only (include/yatt/*.hpp), the way the reference's runner /
// demo worker would call it after the link swap described in INTEGRATION.md.
//
//   1. build the step batch like runner::make_step_batch (runner.cpp:152-166)
//   2. dynamic-sampling rounds for all controller shards on the device
//      (sim::run_rollout_rounds = the shard loop of run_rlhf_step)
//   3. repack accepted lengths into balanced buckets (balancer::sort_and_bucket)
//   4. experience making on the device: logprob/entropy/KL, GRPO advantages,
//      clipped-surrogate + KL loss (experience.hpp), loss finalised on host
//   5. the backward into the logits, the node peer group (world = 1 here),
//      the survivors' payload gather and groups straddling emulated ranks
// Prints a short report and "rank ok"; exits non-zero on any mismatch.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "yatt/balancer.hpp"
#include "yatt/errors.hpp"
#include "yatt/experience.hpp"
#include "yatt/simcore.hpp"
#include "yatt/workload.hpp"
#include "yatt_cuda.h"

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(2);
  }
}

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  ck(cudaMalloc(&p, n * sizeof(T) + 16), "cudaMalloc");
  return static_cast<T*>(p);
}

}  // namespace

int main() {
  using namespace yatt;
  const int prompts = 16, group = 8, T = 256, vocab = 32000, controllers = 4;
  const std::uint64_t seed = 20250814;

  // 1. step batch (sample_id = step * B + i, keyed prompt lengths)
  workload::RolloutBatch batch;
  batch.step_index = 0;
  const workload::LengthDistribution prompt_dist{workload::DistKind::kUniform, 16, 64, 4096};
  for (int i = 0; i < prompts * group; ++i) {
    workload::RolloutSample s;
    s.sample_id = static_cast<std::uint64_t>(i);
    s.prompt_len_tokens = workload::sample_length_keyed(prompt_dist, seed,
                                                        workload::kPromptLenStream, 0, 0,
                                                        s.sample_id);
    batch.samples.push_back(s);
  }

  // 2. dynamic-sampling rounds, every controller shard per launch
  sim::RoundParams params;
  params.out_dist = {workload::DistKind::kUniform, 1, double(T), T};
  params.rejection = {0.3, true, group};
  params.seed = seed;
  params.microbatch_size = 8;
  params.max_rounds = 4;
  const auto rounds = sim::run_rollout_rounds(batch, controllers, params);
  long long units = 0;
  for (const auto& reps : rounds) units += sim::reduce_round_reports(reps).train_units;
  int accepted = 0;
  std::vector<int> lengths;
  for (const auto& s : batch.samples) {
    accepted += s.accepted;
    lengths.push_back(s.prompt_len_tokens + s.target_out_len_tokens);
  }
  std::printf("rollout: %zu rounds, %d/%zu accepted, train_units=%lld\n", rounds.size(), accepted,
              batch.samples.size(), units);
  if (accepted != int(batch.samples.size())) return 1;

  // same rounds from one controller must give the same totals (controller invariance)
  workload::RolloutBatch one = batch;
  for (auto& s : one.samples) s.accepted = false, s.accepted_round = 0, s.target_out_len_tokens = 0;
  long long units1 = 0;
  for (const auto& reps : sim::run_rollout_rounds(one, 1, params))
    units1 += sim::reduce_round_reports(reps).train_units;
  if (units1 != units) {
    std::fprintf(stderr, "controller invariance violated: %lld vs %lld\n", units1, units);
    return 1;
  }

  // 3. balanced repack of the accepted samples
  const balancer::BatchingPlan plan = balancer::sort_and_bucket(lengths, 16, seed);
  const double waste = balancer::padding_waste(plan, lengths);
  std::printf("buckets: %zu, padding waste %.4f (bound %.4f)\n", plan.buckets.size(), waste,
              balancer::waste_bound(16));

  // 4. experience making on the device
  const std::int64_t rows = std::int64_t(prompts) * group * T;
  auto* pol = dalloc<std::uint16_t>(size_t(rows) * vocab);
  auto* ref = dalloc<std::uint16_t>(size_t(rows) * vocab);
  auto* tgt = dalloc<std::int32_t>(size_t(rows));
  auto* stats = dalloc<float>(size_t(rows) * 4);
  auto* rewards = dalloc<float>(size_t(prompts) * group);
  auto* sadv = dalloc<float>(size_t(prompts) * group);
  auto* tadv = dalloc<float>(size_t(rows));
  auto* old = dalloc<float>(size_t(rows));
  auto* cu = dalloc<std::int64_t>(size_t(prompts) * group + 1);
  auto* sums = dalloc<experience::LossSums>(1);
  const size_t ws_bytes = experience::policy_loss_workspace_bytes();
  void* ws = dalloc<std::uint8_t>(ws_bytes);
  detail::throw_status(yatt_synth_logits(seed, 0, rows, vocab, pol, ref, tgt, nullptr));
  detail::throw_status(yatt_synth_floats(seed, 105, 0, prompts * group, YATT_SYNTH_REWARD, group,
                                         nullptr, rewards, nullptr));
  std::vector<std::int64_t> hcu(size_t(prompts) * group + 1);
  for (size_t i = 0; i < hcu.size(); ++i) hcu[i] = std::int64_t(i) * T;
  ck(cudaMemcpy(cu, hcu.data(), hcu.size() * 8, cudaMemcpyHostToDevice), "H2D cu");

  float *logp = stats, *ref_logp = stats + rows, *ent = stats + 2 * rows, *kl = stats + 3 * rows;
  experience::token_logprob_stats(pol, ref, tgt, nullptr, rows, vocab,
                                  experience::KlEstimator::kK3, {logp, ref_logp, ent, kl});
  detail::throw_status(yatt_synth_floats(seed, 104, 0, rows, YATT_SYNTH_OLD_DELTA, 1, logp, old,
                                         nullptr));
  experience::grpo_advantages(rewards, prompts * group, 0, experience::GrpoConfig{group}, sadv);
  detail::throw_status(yatt_broadcast_to_tokens(sadv, cu, prompts * group, nullptr, tadv, rows,
                                                nullptr));
  const experience::PolicyLossConfig cfg;
  experience::policy_loss(logp, old, tadv, kl, ent, nullptr, rows, nullptr, 0, cfg, sums, ws,
                          ws_bytes);
  experience::LossSums h;
  ck(cudaMemcpy(&h, sums, sizeof(h), cudaMemcpyDeviceToHost), "D2H sums");
  const double loss = experience::finalize_loss(h, cfg);
  std::printf("experience: %lld tokens, loss %.6f, mean kl %.6f, mean entropy %.4f, clipfrac %.4f\n",
              (long long)h.token_count, loss, h.kl_sum / h.token_count,
              h.entropy_sum / h.token_count, h.clip_count / h.token_count);
  if (!(h.token_count == double(rows)) || !std::isfinite(loss)) return 1;

  // 5a. backward into the policy logits (first 1,024 rows), rows sum to ~0
  {
    const std::int64_t gr = 1024;
    auto* coef = dalloc<float>(size_t(gr) * 8);
    auto* grad = dalloc<std::uint16_t>(size_t(gr) * vocab);
    experience::policy_logits_grad(pol, ref, tgt, {logp, ref_logp, ent, kl}, old, tadv, nullptr, gr,
                                   vocab, nullptr, 0, cfg, experience::KlEstimator::kK3,
                                   double(rows), coef, grad);
    std::vector<std::uint16_t> hg(static_cast<size_t>(vocab));
    ck(cudaMemcpy(hg.data(), grad, hg.size() * 2, cudaMemcpyDeviceToHost), "D2H grad");
    double sum = 0, amax = 0;
    for (auto b : hg) {
      std::uint32_t u = std::uint32_t(b) << 16;
      float f;
      std::memcpy(&f, &u, 4);
      sum += f;
      amax = std::fmax(amax, std::fabs(f));
    }
    std::printf("backward: row 0 grad sum %.3e (max |g| %.3e)\n", sum, amax);
    if (!std::isfinite(sum) || std::fabs(sum) > 1e-2 * amax * 50) return 1;
    // the fused training-side op (policy logits only, each row read twice):
    // same gradient as the two-kernel path to bf16 rounding
    auto* f_out = dalloc<float>(size_t(gr) * 3);
    auto* grad2 = dalloc<std::uint16_t>(size_t(gr) * vocab);
    experience::policy_loss_grad(pol, nullptr, tgt, nullptr, ref_logp, old, tadv, gr, vocab,
                                 nullptr, 0,
                                 cfg, experience::KlEstimator::kK3, double(rows),
                                 {f_out, nullptr, f_out + gr, f_out + 2 * gr}, grad2);
    std::vector<std::uint16_t> hg2(static_cast<size_t>(vocab));
    ck(cudaMemcpy(hg2.data(), grad2, hg2.size() * 2, cudaMemcpyDeviceToHost), "D2H fused grad");
    int off = 0;
    for (size_t v = 0; v < hg.size(); ++v) {
      float a, b;
      std::uint32_t ua = std::uint32_t(hg[v]) << 16, ub = std::uint32_t(hg2[v]) << 16;
      std::memcpy(&a, &ua, 4);
      std::memcpy(&b, &ub, 4);
      off += !(std::fabs(a - b) <= 0.0079 * std::fabs(a) + 1e-6 * amax);
    }
    std::printf("fused loss+grad: row 0 matches the two-kernel gradient (%d of %d outside bf16)\n",
                off, vocab);
    if (off != 0) return 1;
    cudaFree(f_out);
    cudaFree(grad2);
    cudaFree(coef);
    cudaFree(grad);
  }

  // 5b. peer group (world = 1): the fused reduce + all-reduce == the plain loss
  {
    experience::PeerGroup peer(1, 0);
    peer.connect(peer.handle());
    auto* gsums = dalloc<experience::LossSums>(1);
    peer.policy_loss(logp, old, tadv, kl, ent, nullptr, rows, nullptr, 0, cfg, gsums, ws,
                     ws_bytes);
    experience::LossSums g;
    ck(cudaMemcpy(&g, gsums, sizeof(g), cudaMemcpyDeviceToHost), "D2H peer sums");
    if (std::memcmp(&g, &h, sizeof(g)) != 0 || peer.status() != 0) {
      std::fprintf(stderr, "peer group sums differ from policy_loss\n");
      return 1;
    }
    std::printf("peer group: fused loss all-reduce == policy_loss (bit-exact)\n");
    // all-gather of the round-report words (world 1: the identity)
    std::vector<std::int64_t> hw(100);
    for (int i = 0; i < 100; ++i) hw[size_t(i)] = 7 * i - 3;
    auto* dw = dalloc<std::int64_t>(100);
    auto* dg = dalloc<std::int64_t>(100);
    ck(cudaMemcpy(dw, hw.data(), 800, cudaMemcpyHostToDevice), "H2D words");
    peer.allgather(dw, 100, dg);
    std::vector<std::int64_t> hgw(100);
    ck(cudaMemcpy(hgw.data(), dg, 800, cudaMemcpyDeviceToHost), "D2H gathered");
    if (hgw != hw) return 1;
    cudaFree(dw);
    cudaFree(dg);
    cudaFree(gsums);
    // the one-exchange multi-rank rounds (world 1: this rank holds every
    // sample) == the single-process round loop, report for report
    workload::RolloutBatch fresh = one;
    for (auto& s : fresh.samples) s.accepted = false, s.accepted_round = 0, s.target_out_len_tokens = 0;
    workload::RolloutBatch fresh2 = fresh;
    const auto single = sim::run_rollout_rounds(fresh, 1, params);
    const auto viapeer = peer.run_rollout_rounds(fresh2.samples, fresh2.step_index, params);
    bool same = single.size() == viapeer.size();
    for (size_t r = 0; same && r < single.size(); ++r) {
      const auto& a = single[r][0];
      const auto& b = viapeer[r][0];
      same = a.controller_rank == b.controller_rank && a.round == b.round &&
             a.active_count == b.active_count && a.pending_count == b.pending_count &&
             a.accepted_train_units == b.accepted_train_units &&
             a.microbatches.size() == b.microbatches.size();
    }
    for (size_t i = 0; same && i < fresh.samples.size(); ++i)
      same = fresh.samples[i].target_out_len_tokens == fresh2.samples[i].target_out_len_tokens &&
             fresh.samples[i].accepted_round == fresh2.samples[i].accepted_round;
    if (!same) {
      std::fprintf(stderr, "peer rounds differ from the single-process rounds\n");
      return 1;
    }
    std::printf("peer group: one-exchange rounds == single-process rounds (%zu rounds)\n",
                viapeer.size());
  }

  // 5c. dynamic sampling on the rewards + the survivors' payload in one launch
  {
    const int n = prompts * group;
    auto* lens = dalloc<std::int64_t>(size_t(n));
    std::vector<std::int64_t> hl(static_cast<size_t>(n), T);
    ck(cudaMemcpy(lens, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice), "H2D lens");
    experience::CompactionBuffers plan{dalloc<std::uint8_t>(size_t(n) / group),
                                       dalloc<std::int32_t>(size_t(n)),
                                       dalloc<std::int64_t>(size_t(n) + 1),
                                       dalloc<std::int64_t>(3)};
    const size_t cws_bytes = experience::dynamic_sampling_workspace_bytes(n);
    void* cws = dalloc<std::uint8_t>(cws_bytes);
    experience::dynamic_sampling_filter(rewards, lens, n, group, plan, cws, cws_bytes);
    auto* out_logp = dalloc<float>(size_t(rows));
    auto* out_tgt = dalloc<std::int32_t>(size_t(rows));
    experience::gather_payload({{logp, out_logp, 4}, {tgt, out_tgt, 4}}, cu, plan, n);
    std::int64_t counts[3];
    ck(cudaMemcpy(counts, plan.counts, sizeof(counts), cudaMemcpyDeviceToHost), "D2H counts");
    std::printf("dynamic sampling: %lld of %d samples kept, %lld tokens gathered\n",
                (long long)counts[0], n, (long long)counts[1]);
    if (counts[1] != counts[0] * T) return 1;
  }

  // 5d. groups straddling ranks (sample-level shard_dataset at P = 3): each
  // emulated rank's boundary records, stacked in rank order (what the
  // all-gather delivers), merged on the device -> advantages and the filter's
  // global layout equal the single-rank ones; the peer group's one-call form
  // (world 1) equals the plain op
  {
    const int n = prompts * group, P = 3;
    std::vector<float> one(static_cast<size_t>(n));
    ck(cudaMemcpy(one.data(), sadv, size_t(n) * 4, cudaMemcpyDeviceToHost), "D2H adv");
    auto* lens = dalloc<std::int64_t>(size_t(n));
    std::vector<std::int64_t> hl(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) hl[size_t(i)] = 100 + i % 7;
    ck(cudaMemcpy(lens, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice), "H2D lens");
    auto* grecs = dalloc<double>(size_t(P) * 8);
    auto* frecs = dalloc<std::int64_t>(size_t(P) * 6);
    std::vector<workload::ShardRange> sh;
    std::vector<double*> moms;
    for (int r = 0; r < P; ++r) {
      sh.push_back(workload::shard_dataset(std::uint64_t(n), P, r));
      const std::int64_t b = std::int64_t(sh.back().begin), m = std::int64_t(sh.back().size());
      const std::int64_t ng = experience::grpo_num_local_groups(m, std::uint64_t(b), group);
      moms.push_back(dalloc<double>(size_t(ng) * 3));
      experience::grpo_group_moments(rewards + b, m, std::uint64_t(b), group, moms.back());
      experience::grpo_boundary_record(moms.back(), m, std::uint64_t(b), group, grecs + 8 * r);
      experience::dynamic_sampling_boundary_record(rewards + b, m, std::uint64_t(b), group,
                                                   frecs + 6 * r);
    }
    bool straddles = false;
    std::int64_t kept[3] = {0, 0, 0};
    std::vector<float> got(static_cast<size_t>(n));
    for (int r = 0; r < P; ++r) {
      const std::int64_t b = std::int64_t(sh[size_t(r)].begin);
      const std::int64_t m = std::int64_t(sh[size_t(r)].size());
      straddles = straddles || b % group != 0;
      experience::grpo_merge_boundaries(moms[size_t(r)], m, std::uint64_t(b), group, grecs, P);
      auto* adv_r = dalloc<float>(size_t(m));
      experience::grpo_advantages(rewards + b, m, std::uint64_t(b), experience::GrpoConfig{group},
                                  adv_r, moms[size_t(r)]);
      ck(cudaMemcpy(got.data() + b, adv_r, size_t(m) * 4, cudaMemcpyDeviceToHost), "D2H adv_r");
      const std::int64_t ng = experience::grpo_num_local_groups(m, std::uint64_t(b), group);
      experience::CompactionBuffers pl{dalloc<std::uint8_t>(size_t(ng)),
                                       dalloc<std::int32_t>(size_t(m)),
                                       dalloc<std::int64_t>(size_t(m) + 1),
                                       dalloc<std::int64_t>(3)};
      const size_t wsb = experience::dynamic_sampling_workspace_bytes(m);
      void* w = dalloc<std::uint8_t>(wsb);
      experience::dynamic_sampling_filter_sharded(rewards + b, lens + b, m, std::uint64_t(b),
                                                  group, frecs, P, pl, w, wsb);
      std::int64_t c[3];
      ck(cudaMemcpy(c, pl.counts, sizeof(c), cudaMemcpyDeviceToHost), "D2H counts_r");
      for (int k = 0; k < 3; ++k) kept[k] += c[k];
      cudaFree(adv_r);
      cudaFree(w);
    }
    double worst = 0;
    for (int i = 0; i < n; ++i)
      worst = std::fmax(worst, std::fabs(double(got[size_t(i)]) - double(one[size_t(i)])));
    experience::CompactionBuffers all{dalloc<std::uint8_t>(size_t(n) / group),
                                      dalloc<std::int32_t>(size_t(n)),
                                      dalloc<std::int64_t>(size_t(n) + 1),
                                      dalloc<std::int64_t>(3)};
    const size_t wsb = experience::dynamic_sampling_workspace_bytes(n);
    void* w = dalloc<std::uint8_t>(wsb);
    experience::dynamic_sampling_filter(rewards, lens, n, group, all, w, wsb);
    std::int64_t c1[3];
    ck(cudaMemcpy(c1, all.counts, sizeof(c1), cudaMemcpyDeviceToHost), "D2H counts_1");
    std::printf("straddling groups (P = %d): max |adv - single rank| %.1e, kept %lld/%lld/%lld "
                "(single rank %lld/%lld/%lld)\n", P, worst, (long long)kept[0],
                (long long)kept[1], (long long)kept[2], (long long)c1[0], (long long)c1[1],
                (long long)c1[2]);
    if (!straddles || worst > 1e-6 || std::memcmp(kept, c1, sizeof(c1)) != 0) return 1;
    experience::PeerGroup peer(1, 0);
    peer.connect(peer.handle());
    const size_t pwsb = peer.straddle_workspace_bytes(n, 0, group);
    void* pws = dalloc<std::uint8_t>(pwsb);
    auto* padv = dalloc<float>(size_t(n));
    peer.grpo_advantages(rewards, n, 0, experience::GrpoConfig{group}, padv, pws, pwsb);
    ck(cudaMemcpy(got.data(), padv, size_t(n) * 4, cudaMemcpyDeviceToHost), "D2H peer adv");
    if (std::memcmp(got.data(), one.data(), size_t(n) * 4) != 0) return 1;
    peer.dynamic_sampling_filter(rewards, lens, n, 0, group, all, pws, pwsb);
    ck(cudaMemcpy(c1 + 0, all.counts, sizeof(c1), cudaMemcpyDeviceToHost), "D2H peer counts");
    if (std::memcmp(kept, c1, sizeof(c1)) != 0) return 1;
    for (double* mm : moms) cudaFree(mm);
    cudaFree(w);
    cudaFree(pws);
    cudaFree(padv);
  }

  // errors keep the reference's types
  try {
    balancer::sort_and_bucket(lengths, 0, 1);
    return 1;
  } catch (const ConfigError&) {
  }
  try {
    workload::shard_dataset(10, 3, 3);
    return 1;
  } catch (const RankOutOfRange&) {
  }
  std::printf("rank ok\n");
  return 0;
}
