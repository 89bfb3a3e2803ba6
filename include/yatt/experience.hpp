// yatt/experience.hpp — the experience-making / policy-loss ops (new API).
//
// No counterpart in the reference, where Preparation and Training are cost
// stand-ins (proj/src/simcore.cpp:13-15, :395-406).  Written in the style of
// the reference headers: config structs with validate() throwing ConfigError
// (cf. ControllerTopology::validate, controller.cpp:7-26), exceptions for
// errors.  All pointers are device pointers; every call is stream-ordered on
// `stream` (a cudaStream_t, nullptr = default stream) and does not block.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "yatt/simcore.hpp"

namespace yatt::experience {

// ---- A1 -------------------------------------------------------------------
enum class KlEstimator { kK1 = 0, kK2 = 1, kK3 = 2, kFull = 3 };

struct TokenStats {
  float* logp = nullptr;       // required
  float* ref_logp = nullptr;   // optional outputs may be nullptr
  float* entropy = nullptr;
  float* kl = nullptr;
};

// Row-major [rows, vocab] bf16 logits (uint16 bit patterns); rows with
// mask == 0 are skipped and produce zeros.  vocab % 8 == 0.
void token_logprob_stats(const std::uint16_t* policy_logits, const std::uint16_t* ref_logits,
                         const std::int32_t* targets, const std::uint8_t* mask,
                         std::int64_t rows, int vocab, KlEstimator kl, const TokenStats& out,
                         void* stream = nullptr);

// ---- A2 -------------------------------------------------------------------
struct GrpoConfig {
  int group_size = 8;
  float eps = 1e-6f;
  bool norm_by_std = true;
  void validate() const;
};

// Advantages of n_samples local samples whose global ids start at
// first_sample_id.  group_moments (n, mean, M2 per local group, fp64) may be
// supplied after a cross-rank merge for groups straddling ranks.
void grpo_advantages(const float* rewards, std::int64_t n_samples, std::uint64_t first_sample_id,
                     const GrpoConfig& config, float* advantages,
                     const double* group_moments = nullptr, void* stream = nullptr);

// ---- A3 -------------------------------------------------------------------
struct GaeConfig {
  float gamma = 1.0f;
  float lam = 0.95f;
  void validate() const;
};

// n_tokens = length of the packed arrays; workspace of gae_workspace_bytes(n_tokens).
std::size_t gae_workspace_bytes(std::int64_t n_tokens);
// device_moments (optional, 3 doubles): masked {count, sum, sum_sq} of the
// advantages from the same pass (the whitening statistics).
void gae(const float* values, const float* rewards, const std::uint8_t* mask,
         const std::int64_t* cu_seqlens, std::int64_t n_seqs, std::int64_t n_tokens,
         const GaeConfig& config, float* advantages, float* returns, void* workspace,
         std::size_t workspace_bytes, void* stream = nullptr, double* device_moments = nullptr);

// ---- A4 -------------------------------------------------------------------
enum class LossAggregation { kTokenMean = 0, kSeqMeanTokenMean = 1, kSeqMeanTokenSum = 2 };

struct PolicyLossConfig {
  float clip_low = 0.2f;
  float clip_high = 0.2f;
  float clip_ratio_c = 0.0f;  // dual clip bound (> 1) or 0 = off
  float kl_coef = 0.001f;
  float entropy_coef = 0.0f;
  LossAggregation aggregation = LossAggregation::kTokenMean;
  void validate() const;
};

struct LossSums {  // layout identical to yatt_loss_sums
  double loss_sum = 0, pg_sum = 0, kl_sum = 0, entropy_sum = 0, clip_count = 0, ratio_sum = 0,
         token_count = 0, seq_count = 0;
};

std::size_t policy_loss_workspace_bytes();
void policy_loss(const float* logp, const float* old_logp, const float* advantages,
                 const float* kl, const float* entropy, const std::uint8_t* mask,
                 std::int64_t n_tokens, const std::int64_t* cu_seqlens, std::int64_t n_seqs,
                 const PolicyLossConfig& config, LossSums* device_sums, void* workspace,
                 std::size_t workspace_bytes, void* stream = nullptr);
double finalize_loss(const LossSums& global_sums, const PolicyLossConfig& config);

// Groups straddling ranks (the reference's SAMPLE-level shard_dataset,
// workload.cpp:183-198, with the group unit sample_id / group_size,
// workload.cpp:158-160): the first / last local group of a shard may hold only
// part of a group.  Per-rank moments of the local groups (n, mean, M2; fp64,
// one row per local group); the 8-double boundary record of the first / last
// local group; the merge of every rank's records (gathered in rank order,
// world x 8 doubles) into rows 0 and last — identical bits on every rank.
// Pass the merged moments to grpo_advantages.  PeerGroup::grpo_advantages
// does all of it in one call.
std::int64_t grpo_num_local_groups(std::int64_t n_samples, std::uint64_t first_sample_id,
                                   int group_size);
void grpo_group_moments(const float* rewards, std::int64_t n_samples,
                        std::uint64_t first_sample_id, int group_size, double* moments,
                        void* stream = nullptr);
void grpo_boundary_record(const double* moments, std::int64_t n_samples,
                          std::uint64_t first_sample_id, int group_size, double* record,
                          void* stream = nullptr);
void grpo_merge_boundaries(double* moments, std::int64_t n_samples,
                           std::uint64_t first_sample_id, int group_size,
                           const double* all_records, int world, void* stream = nullptr);

// ---- A5 + A6 --------------------------------------------------------------
struct CompactionBuffers {
  std::uint8_t* keep_groups = nullptr;  // [grpo_num_local_groups(n, first_sample_id, G)]
  std::int32_t* index_map = nullptr;    // [n_samples]
  std::int64_t* new_cu = nullptr;       // [n_samples + 1]
  std::int64_t* counts = nullptr;       // [3] kept samples, tokens, groups
};

std::size_t dynamic_sampling_workspace_bytes(std::int64_t n_samples);
void dynamic_sampling_filter(const float* rewards, const std::int64_t* seq_lens,
                             std::int64_t n_samples, int group_size, const CompactionBuffers& out,
                             void* workspace, std::size_t workspace_bytes,
                             void* stream = nullptr);
// A shard of a sample-level split (global ids from first_sample_id): every
// rank writes its 6-word boundary record ({group, first reward bits,
// any-differs} of its first and last local group); with the records of all
// ranks gathered in rank order (world x 6 int64), every rank holding a piece
// of a straddling group takes the same exact keep decision.  counts[2]
// counts the groups whose first sample is local (each group once globally).
void dynamic_sampling_boundary_record(const float* rewards, std::int64_t n_samples,
                                      std::uint64_t first_sample_id, int group_size,
                                      std::int64_t* record, void* stream = nullptr);
void dynamic_sampling_filter_sharded(const float* rewards, const std::int64_t* seq_lens,
                                     std::int64_t n_samples, std::uint64_t first_sample_id,
                                     int group_size, const std::int64_t* all_records, int world,
                                     const CompactionBuffers& out, void* workspace,
                                     std::size_t workspace_bytes, void* stream = nullptr);

// ---- backward into the policy logits -------------------
// dL/d(policy logits) of the A4 loss as bf16 [rows, vocab].  `stats` are A1's
// outputs (logp, ref_logp, entropy, kl); `norm` = the GLOBAL token count for
// token-mean, the global sequence count for the seq modes (all-reduce first).
// coef: device scratch of 8 floats per row.  ref_logits are read for kFull
// only.  Any vocab; TMA streaming when 16-byte aligned with vocab % 8 == 0.
void policy_logits_grad(const std::uint16_t* policy_logits, const std::uint16_t* ref_logits,
                        const std::int32_t* targets, const TokenStats& stats,
                        const float* old_logp, const float* advantages, const std::uint8_t* mask,
                        std::int64_t rows, int vocab, const std::int64_t* cu_seqlens,
                        std::int64_t n_seqs, const PolicyLossConfig& config, KlEstimator kl,
                        double norm, float* coef, std::uint16_t* grad, void* stream = nullptr);

// ---- training side, fused: loss terms + gradient in one pass pair ----------
// From the policy logits alone: per-token logp / entropy / kl (vs the stored
// ref_logp of the experience stage; nullptr = no KL term) AND the bf16
// gradient dL/d(policy logits); each row is streamed twice, the second read
// from L2 (HBM 4V bytes per row instead of 6V).  kl: kK1 / kK2 / kK3 (vs
// ref_logp; ref_logits may be nullptr) or kFull (reads ref_logits); all
// three aggregations (norm = global valid tokens for token-mean, global
// sequences for the seq modes; seq-mean-token-mean takes cu_seqlens and a
// workspace of policy_loss_grad_workspace_bytes); vocab % 8 == 0, logits and
// grad 16-byte aligned.  out.ref_logp is not written.  The loss sums:
// policy_loss(out.logp, ...).
std::size_t policy_loss_grad_workspace_bytes(std::int64_t rows, LossAggregation aggregation);
void policy_loss_grad(const std::uint16_t* policy_logits, const std::uint16_t* ref_logits,
                      const std::int32_t* targets, const std::uint8_t* mask,
                      const float* ref_logp, const float* old_logp,
                      const float* advantages, std::int64_t rows, int vocab,
                      const std::int64_t* cu_seqlens, std::int64_t n_seqs,
                      const PolicyLossConfig& config, KlEstimator kl, double norm,
                      const TokenStats& out, std::uint16_t* grad, void* workspace = nullptr,
                      std::size_t workspace_bytes = 0, void* stream = nullptr);

// ---- fused LM head + online log-softmax (tcgen05; §8f #4) -------------------
// logp / entropy / lse per row of softmax(hidden @ lm_head^T) without writing
// the logits; hidden [rows, hidden_dim], lm_head [vocab, hidden_dim] bf16.
// n_split: vocabulary splits (1..64), 0 = the library picks (pass the same
// value to lmhead_workspace_bytes).
std::size_t lmhead_workspace_bytes(std::int64_t rows, int vocab, int n_split);
void lmhead_token_stats(const std::uint16_t* hidden, const std::uint16_t* lm_head,
                        const std::int32_t* targets, std::int64_t rows, int hidden_dim, int vocab,
                        int n_split, float* logp, float* entropy, float* lse, void* workspace,
                        std::size_t workspace_bytes, void* stream = nullptr);

// ---- survivors' per-token payload (A6), all arrays in one launch ----------
struct PayloadArray {
  const void* src = nullptr;  // [old_cu[n_samples]] elements
  void* dst = nullptr;        // [kept tokens (+ dst_offset)] elements
  int elem_bytes = 4;         // 1, 2, 4 or 8
};
void gather_payload(const std::vector<PayloadArray>& arrays, const std::int64_t* old_cu,
                    const CompactionBuffers& plan, std::int64_t max_kept,
                    const std::int64_t* dst_offset = nullptr, void* stream = nullptr);

// ---- the node's ranks joined through NVLink peer memory ---------------------
// Construct on every rank, exchange handle() (64 bytes each, rank order) over
// the controller rendezvous, connect().  Collective calls; results are
// bit-identical on all ranks.  No NCCL involved.
class PeerGroup {
 public:
  PeerGroup(int world, int rank);
  ~PeerGroup();
  PeerGroup(const PeerGroup&) = delete;
  PeerGroup& operator=(const PeerGroup&) = delete;
  const std::vector<std::uint8_t>& handle() const { return handle_; }
  void connect(const std::vector<std::uint8_t>& all_handles);
  // out[i] = sum over ranks of in[i], n <= 16 doubles
  void allreduce(const double* in, int n, double* out, void* stream = nullptr);
  // prefix[i] = sum over lower ranks, total[i] = over all ranks (n <= 16)
  void scan(const std::int64_t* in, int n, std::int64_t* prefix, std::int64_t* total,
            void* stream = nullptr);
  // Rank-major all-gather of n <= YATT_PEER_GATHER_MAX_WORDS int64 words
  // (out: world * n), e.g. the round reports + microbatch aggregates.
  void allgather(const std::int64_t* in, int n, std::int64_t* out, void* stream = nullptr);
  // policy_loss whose final reduction is the cross-rank all-reduce: GLOBAL sums
  void policy_loss(const float* logp, const float* old_logp, const float* advantages,
                   const float* kl, const float* entropy, const std::uint8_t* mask,
                   std::int64_t n_tokens, const std::int64_t* cu_seqlens, std::int64_t n_seqs,
                   const PolicyLossConfig& config, LossSums* device_sums, void* workspace,
                   std::size_t workspace_bytes, void* stream = nullptr);
  // Group-level ops of a shard whose first / last groups may straddle ranks
  // (sample-level sharding): boundary record -> peer all-gather -> device
  // merge -> the op, stream-ordered, one call (collective).  Workspace:
  // straddle_workspace_bytes.  Advantages equal a single rank's to fp64
  // rounding of the merged moments; the filter's layout is bit-exact.
  std::size_t straddle_workspace_bytes(std::int64_t n_samples, std::uint64_t first_sample_id,
                                       int group_size) const;
  void grpo_advantages(const float* rewards, std::int64_t n_samples,
                       std::uint64_t first_sample_id, const GrpoConfig& config,
                       float* advantages, void* workspace, std::size_t workspace_bytes,
                       void* stream = nullptr);
  void dynamic_sampling_filter(const float* rewards, const std::int64_t* seq_lens,
                               std::int64_t n_samples, std::uint64_t first_sample_id,
                               int group_size, const CompactionBuffers& out, void* workspace,
                               std::size_t workspace_bytes, void* stream = nullptr);
  // The multi-rank dynamic-sampling step with ONE exchange
  // (yatt_peer_rounds_run): this rank's controller shard (the reference's
  // shard_dataset range, workload.cpp:183-198) runs every round in one
  // persistent kernel and every rank's reports travel once; returns the
  // GLOBAL reports[round][rank] (what the reference's coordinator feeds to
  // StepAssembler::feed_round, demo.cpp:468-476) and updates the shard's
  // samples like copy_back (simcore.cpp:107-119).  Collective.
  std::vector<std::vector<sim::ShardRoundReport>> run_rollout_rounds(
      std::vector<workload::RolloutSample>& shard_samples, int step_index,
      const sim::RoundParams& params, std::vector<int>* first_round_lengths = nullptr);
  int world() const { return world_; }
  int rank() const { return rank_; }
  int status() const;  // 1 after a call timed out waiting for a rank

 private:
  void* h_ = nullptr;
  std::vector<std::uint8_t> handle_;
  int world_ = 0, rank_ = 0;
};

}  // namespace yatt::experience
