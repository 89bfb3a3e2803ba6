// run_rlhf_step.cpp — drop-in definition of yatt::sim::run_rlhf_step
// (reference proj/src/simcore.cpp:462-494) for the integration build.
//
// Compiled into the reference-side binary (INTEGRATION.md §2,
// oracle/Makefile `simcore_b200`), not into libyatt_b200.so: it needs the
// reference's timing layer (StepAssembler, cluster / placement headers),
// which stays the reference's own code.  What changes is the data plane:
// the reference calls shard_round_output once per shard per round and
// feeds each round's reports to the assembler; here ONE device call
// (sim::run_rollout_rounds -> yatt_rounds_run: a persistent kernel over
// every shard and every round, continue test on the device) produces all
// rounds' reports, which are then fed to the unchanged StepAssembler in the
// same order — so the trace is the reference's trace.
#include <vector>

#include "yatt/errors.hpp"
#include "yatt/simcore.hpp"

#ifndef YATT_HAS_TIMING_LAYER
#error "build with the reference's include directory after this repo's (see INTEGRATION.md)"
#endif

namespace yatt::sim {

StepResult run_rlhf_step(const placement::PlacementPlan& plan, workload::RolloutBatch& batch,
                         const StepContext& ctx) {
  // Same validation, same order, same exceptions (simcore.cpp:464-466).
  ctx.out_dist.validate();
  if (ctx.max_rounds < 1) throw ConfigError("max_rounds must be at least 1");
  if (ctx.num_controllers < 1) throw ConfigError("num_controllers must be positive");
  const RoundParams params{ctx.out_dist, ctx.rejection, ctx.seed, ctx.microbatch_size,
                           ctx.max_rounds};
  // The reference's assembler validates the plan / cluster before any round
  // runs (its constructor, simcore.cpp:271-285); keep that order of errors.
  StepAssembler assembler(plan, ctx, batch.step_index);
  if (params.microbatch_size <= 0) throw ConfigError("microbatch_size must be positive");

  std::vector<int> first_lengths;
  const auto rounds = run_rollout_rounds(batch, ctx.num_controllers, params, &first_lengths);

  StepResult result;
  // Round-1 snapshot per controller shard (capture_snapshot, simcore.cpp:122-136).
  result.snapshot.num_controllers = ctx.num_controllers;
  for (int r = 0; r < ctx.num_controllers; ++r) {
    const workload::ShardRange range = workload::shard_dataset(
        static_cast<std::uint64_t>(batch.samples.size()), ctx.num_controllers, r);
    std::vector<std::pair<int, int>> lengths;
    lengths.reserve(range.size());
    for (std::uint64_t i = range.begin; i < range.end; ++i)
      lengths.emplace_back(batch.samples[i].prompt_len_tokens, first_lengths[i]);
    result.snapshot.shard_lengths.push_back(std::move(lengths));
  }
  for (const auto& reports : rounds)
    if (!assembler.feed_round(reports)) break;
  result.trace = assembler.finish();
  return result;
}

}  // namespace yatt::sim
