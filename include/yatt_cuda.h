/*
 * yatt_cuda.h — C ABI of the B200 experience-making path.
 *
 * This is the drop-in boundary between a WeChat-YATT parallel-controller
 * rank (host, C++) and the sm_100a kernels.  Every entry point takes plain
 * pointers + explicit sizes, returns an int status (YATT_OK == 0) and never
 * throws.  The C++ wrappers in include/yatt/*.hpp map the status codes back
 * onto the reference's exception types (reference proj/include/yatt/
 * errors.hpp:10-48) so callers written against the reference keep working.
 *
 * Conventions
 *  - `d_` pointers are device pointers, `h_` pointers host pointers.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - All device work is stream-ordered; a function only synchronises when it
 *    returns host data (documented per function).
 *  - bf16 tensors are passed as uint16_t bit patterns.
 *  - Reentrant given distinct buffers and streams; the last-error message is
 *    thread-local.
 *  - Every pointer must be naturally aligned for its element type (structs:
 *    8 bytes; workspaces: 8, the LM-head one 16); the logits-backward `coef`
 *    table and synth_logits outputs need 16 bytes.
 *    A misaligned pointer returns YATT_ERR_CONFIG before any launch.
 *    yatt_token_stats and yatt_logits_backward accept any vocab and 2-byte
 *    aligned logits (a generic element-wise kernel; the TMA path otherwise).
 *  - Targets must lie in [0, vocab).  A target outside it (device data, so
 *    not checked on the host) never causes an out-of-row access: that row's
 *    logp / ref_logp / kl come out NaN (entropy stays valid) and its
 *    gradient row is NaN, so the error is visible in the outputs.
 */
#ifndef YATT_CUDA_H_
#define YATT_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* Status codes and errors                                                   */
/* ------------------------------------------------------------------------ */
enum yatt_status {
  YATT_OK = 0,
  YATT_ERR_CONFIG = 1,        /* -> yatt::ConfigError          (errors.hpp:45) */
  YATT_ERR_RANK = 2,          /* -> yatt::RankOutOfRange       (errors.hpp:25) */
  YATT_ERR_DISTRIBUTION = 3,  /* -> yatt::InvalidDistribution  (errors.hpp:20) */
  YATT_ERR_CUDA = 4,          /* -> yatt::Error (fail-fast)                    */
  YATT_ERR_NCCL = 5,          /* -> yatt::Error                                */
  YATT_ERR_WORKSPACE = 6      /* workspace too small -> yatt::ConfigError      */
};

/* Message for the last non-OK status returned on this thread. */
const char* yatt_last_error_message(void);
/* ABI version: bumped on any signature change. */
int yatt_abi_version(void);
/* Name of the device the library runs on ("" if none); sm major/minor. */
int yatt_device_info(int device, char* name, int name_len, int* sm_major,
                     int* sm_minor, int* num_sms);

/* ------------------------------------------------------------------------ */
/* Shared POD types (mirror proj/include/yatt/{workload,simcore}.hpp)        */
/* ------------------------------------------------------------------------ */
enum yatt_dist_kind {           /* workload.hpp:10-15 DistKind */
  YATT_DIST_CONSTANT = 0,
  YATT_DIST_UNIFORM = 1,
  YATT_DIST_NORMAL = 2,
  YATT_DIST_LOGNORMAL = 3
};

typedef struct yatt_length_dist {  /* workload.hpp:25-36 LengthDistribution */
  int32_t kind;
  int32_t max_len_tokens;
  double p1;
  double p2;
} yatt_length_dist;

typedef struct yatt_rejection_config {  /* workload.hpp:73-80 RejectionConfig */
  double reject_rate;
  int32_t per_group;
  int32_t group_size;
} yatt_rejection_config;

typedef struct yatt_round_params {  /* simcore.hpp:93-99 RoundParams */
  yatt_length_dist out_dist;
  yatt_rejection_config rejection;
  uint64_t seed;
  int32_t microbatch_size;
  int32_t max_rounds;
} yatt_round_params;

/* One sample of a controller shard: simcore.hpp:78-84 ShardSampleState and
 * workload.hpp:38-46 RolloutSample share this 24-byte device layout. */
typedef struct yatt_sample {
  uint64_t sample_id;
  int32_t prompt_len_tokens;
  int32_t out_len_tokens;
  int32_t accepted_round;
  int32_t accepted;  /* 0/1 */
} yatt_sample;

typedef struct yatt_mb_agg {  /* simcore.hpp:55-62 MicrobatchAggregate */
  int32_t controller_rank;
  int32_t mb_index;
  int32_t sample_count;
  int32_t max_out_len_tokens;
  int64_t score_tokens;
} yatt_mb_agg;

typedef struct yatt_round_report {  /* simcore.hpp:64-76 ShardRoundReport */
  int32_t controller_rank;
  int32_t round;
  int32_t active_count;
  int32_t newly_accepted_count;
  int32_t forced_accept_count;
  int32_t pending_count;
  int64_t accepted_score_tokens;
  int64_t accepted_train_units;
  int64_t num_microbatches;  /* entries written to the microbatch array */
} yatt_round_report;

/* ------------------------------------------------------------------------ */
/* R1  shard_dataset  (replaces workload.cpp:183-198; host, O(1))            */
/* ------------------------------------------------------------------------ */
int yatt_shard_dataset(uint64_t total_samples, int32_t num_controllers,
                       int32_t controller_rank, uint64_t* h_begin,
                       uint64_t* h_end);

/* ------------------------------------------------------------------------ */
/* R6  keyed length draws  (replaces workload.cpp:109-132 batched)           */
/* out[i] = sample_length_keyed(dist, seed, stream_id, step, round, ids[i]). */
/* ------------------------------------------------------------------------ */
int yatt_sample_lengths_keyed(const yatt_length_dist* dist, uint64_t seed,
                              uint64_t stream_id, uint64_t step, uint64_t round,
                              const uint64_t* d_sample_ids, int64_t n,
                              int32_t* d_out, void* stream);

/* ------------------------------------------------------------------------ */
/* R5  rejection_process  (replaces workload.cpp:145-167)                    */
/* d_rejected[i] = 1 iff sample i is pending and its keyed draw < rate.      */
/* ------------------------------------------------------------------------ */
int yatt_rejection_flags(const yatt_sample* d_samples, int64_t n,
                         int32_t step_index, int32_t round,
                         const yatt_rejection_config* config, uint64_t seed,
                         uint8_t* d_rejected, void* stream);

/* ------------------------------------------------------------------------ */
/* R3+R4  shard_round_output  (replaces simcore.cpp:157-214 + :17-39)        */
/* One round of `num_shards` controller shards, device-resident: the        */
/* building block of the multi-rank loop (reports are exchanged between      */
/* ranks before the continue test; ranks.exchange_round_reports).            */
/* Shard s owns d_samples[h_shard_offsets[s] .. h_shard_offsets[s+1]) (host  */
/* array, num_shards+1 entries) and has controller rank first_rank + s.      */
/* Samples are mutated in place exactly like ShardState; the report of       */
/* shard s goes to d_reports[s]; its microbatches to d_mbs + M_s where       */
/* M_s = sum_{s'<s} ceil(n_s' / microbatch_size) (capacity per shard is      */
/* ceil(n_s / microbatch_size); report.num_microbatches are valid).          */
/* ------------------------------------------------------------------------ */
int yatt_shard_round(yatt_sample* d_samples, const int64_t* h_shard_offsets,
                     int32_t num_shards, int32_t first_rank,
                     int32_t step_index, int32_t round,
                     const yatt_round_params* params,
                     yatt_round_report* d_reports, yatt_mb_agg* d_mbs,
                     void* stream);

/* R8  integer part of StepAssembler::feed_round (simcore.cpp:304-311) on the */
/* device, over n reports (all ranks' reports after an all-gather of the     */
/* 48-byte structs = the binary wire format replacing demo.cpp:32-76):       */
/* d_out[6] = {sum active, sum pending, sum forced, sum train_units,          */
/*             sum score_tokens, continue (= sum pending > 0)}.              */
int yatt_reduce_round_reports(const yatt_round_report* d_reports, int32_t n,
                              int64_t* d_out, void* stream);

/* ------------------------------------------------------------------------ */
/* R3+R4+R8  the whole round loop of one step, host buffers                  */
/* (replaces run_rlhf_step's loop simcore.cpp:470-490 over                   */
/* shard_round_output :157-214 + feed_round's continue test :304-311, :382;  */
/* with round_limit = 1, one shard_round_output call).                       */
/*                                                                           */
/*   yatt_rounds_stage   pinned, device-mapped SoA arrays for n samples of   */
/*                       num_shards shards; the caller fills sample_id,      */
/*                       prompt_len and accepted (1 = accepted before the    */
/*                       call: never touched)                                */
/*   yatt_rounds_run     rounds first_round.. of every shard until no sample */
/*                       is pending (or round_limit rounds; <= 0: no limit): */
/*                       ONE persistent kernel reads the stage over PCIe,    */
/*                       takes the continue test on the device and stores    */
/*                       its results straight into the stage; one launch,    */
/*                       one synchronize                                     */
/*   yatt_rounds_result  reports / microbatches (valid until the next run)   */
/*                                                                           */
/* Outputs for samples pending at the start of the call: out_len,            */
/* accepted_round, accepted_out and (if asked) first_round_len = out_len     */
/* after first_round (the run_rlhf_step snapshot); entries of samples        */
/* accepted before the call are placeholders.                                */
/* Shard s owns samples [h_shard_offsets[s], h_shard_offsets[s+1]) with      */
/* controller rank first_rank + s.  Reports are round-major:                 */
/* reports[r * num_shards + s]; microbatches are concatenated in (round,     */
/* shard, mb_index) order, reports[.].num_microbatches of them per report.   */
/* Normal / LogNormal draws the device cannot certify equal to glibc's       */
/* (within 1e-9 relative of a .5 rounding tie) are recomputed on the host    */
/* with glibc and the launch is re-run with them: bit-exact by construction  */
/* (redrawn_on_host counts them).  One handle per thread; the handle belongs */
/* to the device current at create.                                          */
/* ------------------------------------------------------------------------ */
typedef struct yatt_rounds* yatt_rounds_t;

typedef struct yatt_rounds_io {
  uint64_t* sample_id;       /* in  */
  int32_t* prompt_len;       /* in  */
  uint8_t* accepted;         /* in  */
  int32_t* out_len;          /* out */
  int32_t* accepted_round;   /* out */
  uint8_t* accepted_out;     /* out */
  int32_t* first_round_len;  /* out (want_first_round_lens) */
} yatt_rounds_io;

typedef struct yatt_rounds_view {
  const yatt_round_report* reports;    /* rounds * num_shards */
  int32_t rounds;
  int32_t num_shards;
  const yatt_mb_agg* microbatches;
  int64_t num_microbatches;
  int64_t redrawn_on_host;
  int32_t first_round_lens_valid;
} yatt_rounds_view;

int yatt_rounds_create(yatt_rounds_t* out);
void yatt_rounds_destroy(yatt_rounds_t h);
int yatt_rounds_stage(yatt_rounds_t h, int64_t n, int32_t num_shards,
                      yatt_rounds_io* io);
int yatt_rounds_run(yatt_rounds_t h, int64_t n, const int64_t* h_shard_offsets,
                    int32_t num_shards, int32_t first_rank, int32_t step_index,
                    int32_t first_round, int32_t round_limit,
                    const yatt_round_params* params, int32_t want_first_round_lens,
                    void* stream);
int yatt_rounds_result(yatt_rounds_t h, yatt_rounds_view* out);

/* Keyed length draws for HOST ids/out (R6, workload.cpp:109-132), bit-exact */
/* by construction for every distribution (uncertified Normal / LogNormal    */
/* draws are redone with glibc).  Blocks.                                    */
int yatt_sample_lengths_host(const yatt_length_dist* dist, uint64_t seed,
                             uint64_t stream_id, uint64_t step, uint64_t round,
                             const uint64_t* h_sample_ids, int64_t n,
                             int32_t* h_out);

/* Certification band of the Normal / LogNormal device draws (default 1e-9, */
/* relative).  Tests widen it to force the glibc re-draw path.              */
int yatt_set_tie_band(double band);

/* Draws of the device-resident entry points (yatt_sample_lengths_keyed,   */
/* yatt_shard_round) that were NOT certified equal to glibc since the last */
/* reset (their device value was used).  Synchronizes the device.           */
int yatt_uncertified_draws(int64_t* h_count, int32_t reset);

/* ------------------------------------------------------------------------ */
/* A1  fused token statistics over policy + reference logits                 */
/* For each row r (token) of the row-major [rows, vocab] bf16 tensors:       */
/*   logp[r]     = log softmax(policy[r])[target[r]]                         */
/*   ref_logp[r] = log softmax(ref[r])[target[r]]                            */
/*   entropy[r]  = H(softmax(policy[r]))                                     */
/*   kl[r]       = per kl_mode (Delta = ref_logp - logp):                    */
/*       K1: -Delta   K2: Delta^2/2   K3: exp(Delta) - Delta - 1             */
/*       FULL: sum_v p_v (log p_v - log q_v)                                 */
/* Rows with d_mask[r] == 0 (d_mask may be NULL = all valid) are not read    */
/* and produce zeros.  Any vocab size / alignment; vocab % 8 == 0 with      */
/* 16-byte aligned tensors takes the TMA streaming path, others a generic   */
/* scalar-load path with identical results.                                 */
/* Any output pointer may be NULL except d_logp.                             */
/* ------------------------------------------------------------------------ */
enum yatt_kl_mode { YATT_KL_K1 = 0, YATT_KL_K2 = 1, YATT_KL_K3 = 2, YATT_KL_FULL = 3 };

int yatt_token_stats(const uint16_t* d_policy_logits,
                     const uint16_t* d_ref_logits, const int32_t* d_targets,
                     const uint8_t* d_mask, int64_t rows, int32_t vocab,
                     int32_t kl_mode, float* d_logp, float* d_ref_logp,
                     float* d_entropy, float* d_kl, void* stream);

/* Same op, HOST buffers (pageable or pinned): the e2e path.  Streams the    */
/* rows through device staging buffers in chunks, overlapping H2D copies of  */
/* chunk i+1 with the kernel on chunk i, and copies outputs back.  Blocks    */
/* until the outputs are on the host.                                        */
int yatt_token_stats_host(const uint16_t* h_policy_logits,
                          const uint16_t* h_ref_logits,
                          const int32_t* h_targets, const uint8_t* h_mask,
                          int64_t rows, int32_t vocab, int32_t kl_mode,
                          float* h_logp, float* h_ref_logp, float* h_entropy,
                          float* h_kl);

/* ------------------------------------------------------------------------ */
/* A2  GRPO group advantages                                                 */
/* Groups are runs of `group_size` consecutive GLOBAL sample ids; the local  */
/* samples start at global id `first_sample_id`.  Per group g:               */
/*   mean_g, M2_g (two-pass, fp64); std_g = sqrt(M2_g/(n_g-1)) (n_g > 1)     */
/*   adv_i = (r_i - mean_g) / (std_g + eps)   if norm_by_std                 */
/*   adv_i = (r_i - mean_g)                   otherwise                      */
/* n_g == 1 -> adv = 0.  Group moments are (n, mean, M2) triples in fp64.    */
/* Straddling groups (multi-rank): compute local moments with               */
/* yatt_grpo_group_moments, exchange/merge (Chan et al.), then pass the     */
/* merged table to yatt_grpo_advantages via d_group_moments.                 */
/* ------------------------------------------------------------------------ */
int64_t yatt_grpo_num_local_groups(int64_t n_samples, uint64_t first_sample_id,
                                   int32_t group_size);
int yatt_grpo_group_moments(const float* d_rewards, int64_t n_samples,
                            uint64_t first_sample_id, int32_t group_size,
                            double* d_group_moments /* [n_local_groups*3] */,
                            void* stream);
int yatt_grpo_advantages(const float* d_rewards, int64_t n_samples,
                         uint64_t first_sample_id, int32_t group_size,
                         float eps, int32_t norm_by_std,
                         const double* d_group_moments /* NULL: compute */,
                         float* d_sample_adv, void* stream);
/* Boundary exchange for straddling groups, on the device: this rank's      */
/* 8-double record {group, n, mean, M2} x {first, last local group}; after   */
/* an all-gather of every rank's record (world x 8, rank order), the merge   */
/* replaces rows 0 and n_local-1 of the moments table with the Chan merge    */
/* of all pieces of those groups (same order on every rank: identical bits). */
int yatt_grpo_boundary_record(const double* d_group_moments, int64_t n_samples,
                              uint64_t first_sample_id, int32_t group_size,
                              double* d_record /* [8] */, void* stream);
int yatt_grpo_merge_boundaries(double* d_group_moments, int64_t n_samples,
                               uint64_t first_sample_id, int32_t group_size,
                               const double* d_all_records, int32_t world,
                               void* stream);
/* Broadcast one value per sample over its tokens: out[t] = val[s(t)]*mask[t] */
/* where sample s owns tokens [cu[s], cu[s+1]).  d_mask may be NULL.         */
int yatt_broadcast_to_tokens(const float* d_sample_vals,
                             const int64_t* d_cu_seqlens, int64_t n_samples,
                             const uint8_t* d_mask, float* d_token_vals,
                             int64_t n_tokens, void* stream);

/* ------------------------------------------------------------------------ */
/* A3  PPO GAE over packed variable-length sequences                         */
/* Sequence s owns tokens [cu[s], cu[s+1]).  Reverse recursion per sequence  */
/* over valid (mask != 0) tokens; masked tokens are transparent (carry the   */
/* running value and advantage, emit the carried advantage):                 */
/*   delta_t = r_t + gamma * V_next - V_t   (V_next = 0 past the end)        */
/*   A_t     = delta_t + gamma*lam * A_next ;  R_t = A_t + V_t               */
/* Computed in fp64 on the device, stored fp32.  d_mask may be NULL.         */
/* n_tokens: length of the packed arrays (tokens outside [cu[0], cu[n_seqs]) */
/* are not written).  One pass over the tokens: a tiled scan whose tiles    */
/* exchange carries through the workspace (yatt_gae_workspace_bytes).       */
/* ------------------------------------------------------------------------ */
size_t yatt_gae_workspace_bytes(int64_t n_tokens);
int yatt_gae(const float* d_values, const float* d_rewards,
             const uint8_t* d_mask, const int64_t* d_cu_seqlens,
             int64_t n_seqs, int64_t n_tokens, float gamma, float lam,
             float* d_advantages, float* d_returns, void* d_workspace,
             size_t workspace_bytes, void* stream);
/* yatt_gae that also writes the masked moments {count, sum, sum_sq} of the   */
/* advantages it stores (the whitening statistics of yatt_masked_moments,     */
/* accumulated in the same pass; same workspace).                            */
int yatt_gae_with_moments(const float* d_values, const float* d_rewards,
                          const uint8_t* d_mask, const int64_t* d_cu_seqlens,
                          int64_t n_seqs, int64_t n_tokens, float gamma, float lam,
                          float* d_advantages, float* d_returns, double* d_moments,
                          void* d_workspace, size_t workspace_bytes, void* stream);
/* Masked moments {count, sum, sum_sq} (fp64, deterministic) of x, written    */
/* to d_out[3]; all-reduce them across ranks before yatt_whiten.             */
size_t yatt_masked_moments_workspace_bytes(void);
int yatt_masked_moments(const float* d_x, const uint8_t* d_mask, int64_t n,
                        double* d_out, void* d_workspace, size_t workspace_bytes,
                        void* stream);
/* x <- (x - mean) * rsqrt(var + 1e-8) (+ mean if !shift_mean), masked      */
/* tokens untouched; var is unbiased.                                        */
int yatt_whiten(float* d_x, const uint8_t* d_mask, int64_t n,
                const double* d_moments, int32_t shift_mean, void* stream);

/* ------------------------------------------------------------------------ */
/* A4  fused clipped-surrogate + KL-penalty loss, masked token sums          */
/*   ratio = exp(logp - old_logp)                                            */
/*   pg    = max(-A*ratio, -A*clip(ratio, 1-clip_low, 1+clip_high))          */
/*   if clip_ratio_c > 1 and A < 0: pg = min(pg, -A*clip_ratio_c) (dual clip)*/
/*   L_t   = pg + kl_coef*kl_t - entropy_coef*H_t                            */
/* Writes one yatt_loss_sums (fp64, deterministic order) to d_sums.  The     */
/* global token-mean loss is sums.loss_sum / sums.token_count after the      */
/* cross-rank all-reduce (yatt_loss_finalize).                               */
/* ------------------------------------------------------------------------ */
typedef struct yatt_loss_config {
  float clip_low;      /* eps_low, e.g. 0.2 */
  float clip_high;     /* eps_high, e.g. 0.2 (DAPO clip-higher 0.28) */
  float clip_ratio_c;  /* dual-clip bound (>1) or 0 = off */
  float kl_coef;       /* beta */
  float entropy_coef;
  int32_t agg_mode;    /* 0 token-mean, 1 seq-mean-token-mean, 2 seq-mean-token-sum */
} yatt_loss_config;

typedef struct yatt_loss_sums {
  double loss_sum;       /* sum_t m_t L_t  (agg_mode 0) or sum_s seq-term   */
  double pg_sum;         /* sum_t m_t pg_t                                  */
  double kl_sum;         /* sum_t m_t kl_t                                  */
  double entropy_sum;    /* sum_t m_t H_t                                   */
  double clip_count;     /* sum_t m_t [clipped]                             */
  double ratio_sum;      /* sum_t m_t ratio_t                               */
  double token_count;    /* sum_t m_t                                       */
  double seq_count;      /* sequences with >= 1 valid token (modes 1, 2)    */
} yatt_loss_sums;

size_t yatt_policy_loss_workspace_bytes(int64_t n_tokens, int64_t n_seqs,
                                        int32_t agg_mode);
int yatt_policy_loss(const float* d_logp, const float* d_old_logp,
                     const float* d_advantages, const float* d_kl,
                     const float* d_entropy, const uint8_t* d_mask,
                     int64_t n_tokens, const int64_t* d_cu_seqlens,
                     int64_t n_seqs, const yatt_loss_config* config,
                     yatt_loss_sums* d_sums, void* d_workspace,
                     size_t workspace_bytes, void* stream);
/* Host: final scalar loss from (all-reduced) sums. */
double yatt_loss_finalize(const yatt_loss_sums* h_sums,
                          const yatt_loss_config* config);

/* One GRPO experience step from HOST buffers (the e2e plugin call): rows =  */
/* n_samples * T tokens (T = rows / n_samples per sample, sample-major),     */
/* logits streamed H2D in chunks overlapped with A1, then GRPO advantages    */
/* (groups of group_size samples, global ids from first_sample_id), token    */
/* broadcast and the A4 loss; writes the 8 loss sums to h_sums and, if       */
/* non-NULL, the per-token stats to h_stats [4][rows] (logp, ref_logp,       */
/* entropy, kl).  Blocks until h_sums is valid.                              */
int yatt_grpo_step_host(const uint16_t* h_policy_logits,
                        const uint16_t* h_ref_logits, const int32_t* h_targets,
                        const uint8_t* h_mask, int64_t rows, int32_t vocab,
                        const float* h_rewards, int64_t n_samples,
                        uint64_t first_sample_id, int32_t group_size,
                        const float* h_old_logp, const yatt_loss_config* config,
                        int32_t kl_mode, yatt_loss_sums* h_sums, float* h_stats);

/* ------------------------------------------------------------------------ */
/* Fused LM-head GEMM + online log-softmax on tcgen05     */
/* logits = hidden[rows, hidden] . lm_head[vocab, hidden]^T (bf16, fp32       */
/* accumulate in TMEM) are never materialised; per row writes               */
/* logp (target log-prob), entropy and lse (any output but logp may be      */
/* NULL).  n_split splits the vocabulary across CTAs (1..64) to fill the    */
/* GPU when rows are few (0: the library picks; pass the same value to      */
/* yatt_lmhead_workspace_bytes); hidden % 8 == 0; operands 16-B aligned.     */
/* Run once per model (policy, reference) then yatt_kl_from_logps.           */
/* ------------------------------------------------------------------------ */
size_t yatt_lmhead_workspace_bytes(int64_t rows, int32_t vocab, int32_t n_split);
int yatt_lmhead_token_stats(const uint16_t* d_hidden, const uint16_t* d_lm_head,
                            const int32_t* d_targets, int64_t rows,
                            int32_t hidden, int32_t vocab, int32_t n_split,
                            float* d_logp, float* d_entropy, float* d_lse,
                            void* d_workspace, size_t workspace_bytes,
                            void* stream);
/* kl[i] from token log-probs (K1 / K2 / K3; Delta = ref_logp - logp). */
int yatt_kl_from_logps(const float* d_logp, const float* d_ref_logp, int64_t n,
                       int32_t kl_mode, float* d_kl, void* stream);

/* ------------------------------------------------------------------------ */
/* Backward into the policy logits                        */
/* Per token t: dL/dx_v = g (1[v=y] - p_v) + h p_v (log p_v + H)              */
/*                        + f p_v (log p_v - log q_v - KL)                   */
/* for the loss of yatt_policy_loss with the same config and kl_mode.        */
/* Step 1: per-token coefficients (8 floats/token: g, h, f, lse_p, lse_q, H,  */
/* KL, scratch); `norm` = the GLOBAL normaliser after the all-reduce:        */
/* token_count (token-mean) or seq_count (seq-mean modes).  FULL KL needs     */
/* the reference logits + ref_logp; other modes may pass NULL for them.      */
/* Step 2: stream the policy logits (+ reference for FULL) and write the     */
/* gradient as bf16 [rows, vocab]; masked rows get zeros.                    */
/* ------------------------------------------------------------------------ */
int yatt_policy_grad_coef(const uint16_t* d_policy_logits,
                          const uint16_t* d_ref_logits, const int32_t* d_targets,
                          const float* d_logp, const float* d_ref_logp,
                          const float* d_old_logp, const float* d_advantages,
                          const float* d_entropy, const float* d_kl,
                          const uint8_t* d_mask, int64_t n_tokens, int32_t vocab,
                          const int64_t* d_cu_seqlens, int64_t n_seqs,
                          const yatt_loss_config* config, int32_t kl_mode,
                          double norm, float* d_coef, void* stream);
int yatt_logits_backward(const uint16_t* d_policy_logits,
                         const uint16_t* d_ref_logits, const int32_t* d_targets,
                         const uint8_t* d_mask, int64_t rows, int32_t vocab,
                         const float* d_coef, int32_t full_kl, uint16_t* d_grad,
                         void* stream);

/* Training side, fused: the policy loss terms AND d(loss)/d(policy logits)  */
/* in one kernel (A1 on the policy logits only + A4's per-token coefficients */
/* + the backward above).  Each row is streamed twice, the second read from  */
/* L2: HBM bytes 2V read + 2V written per row instead of 6V for              */
/* yatt_token_stats (policy only) + yatt_logits_backward.  The reference     */
/* log-probs come from the experience stage (d_ref_logp, per token; NULL =   */
/* no KL term).  kl_mode K1/K2/K3 use d_ref_logp (d_ref_logits may be NULL);*/
/* kl_mode FULL reads d_ref_logits (same layout as the policy) in both      */
/* passes.  All three aggregations: norm = the global                       */
/* valid-token count (token-mean) or the global sequence count (seq modes);  */
/* seq-mean-token-mean also needs d_cu_seqlens and a workspace of           */
/* yatt_policy_loss_grad_workspace_bytes (per-token scale; 0 bytes for the   */
/* other modes).  vocab % 8 == 0, logits and grad 16-byte aligned.  Writes   */
/* per-token logp / entropy / kl (entropy, kl may be NULL) and grad          */
/* [rows, vocab] bf16 (zero rows where mask == 0); the loss sums follow from */
/* yatt_policy_loss on those per-token outputs.                              */
/* Replaces: Train stand-in simcore.cpp:404-406 (new).          */
size_t yatt_policy_loss_grad_workspace_bytes(int64_t rows, int32_t agg_mode);
int yatt_policy_loss_grad(const uint16_t* d_policy_logits,
                          const uint16_t* d_ref_logits, const int32_t* d_targets,
                          const uint8_t* d_mask, const float* d_ref_logp,
                          const float* d_old_logp, const float* d_advantages,
                          int64_t rows, int32_t vocab, const int64_t* d_cu_seqlens,
                          int64_t n_seqs, const yatt_loss_config* config,
                          int32_t kl_mode, double norm, float* d_logp,
                          float* d_entropy, float* d_kl, uint16_t* d_grad,
                          void* d_workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* A5+A6  dynamic-sampling filter and compaction (bit-exact)                 */
/* keep_g = !(all rewards of group g are bitwise identical).  Groups are     */
/* `group_size` consecutive sample ids; yatt_filter_compact takes a batch    */
/* starting at id 0 (a trailing partial group is a group of its own).        */
/* Survivors keep sample order:                                              */
/*   d_index_map[j] = local index of the j-th kept sample                    */
/*   d_new_cu[j]    = packed token start of kept sample j (local, from 0);   */
/*                    d_new_cu[n_kept] = kept tokens                         */
/*   d_counts[3]    = {kept_samples, kept_tokens, kept_groups}               */
/* Everything stays on the device (no host sync).  For a global packed       */
/* layout across ranks: all-gather d_counts, yatt_exclusive_offset -> the    */
/* rank's token/sample offset, pass it as d_dst_offset to the gathers.       */
/* ------------------------------------------------------------------------ */
size_t yatt_filter_compact_workspace_bytes(int64_t n_samples);
int yatt_filter_compact(const float* d_rewards, const int64_t* d_seq_lens,
                        int64_t n_samples, int32_t group_size,
                        uint8_t* d_keep_groups, int32_t* d_index_map,
                        int64_t* d_new_cu, int64_t* d_counts, void* d_workspace,
                        size_t workspace_bytes, void* stream);
/* Sharded form (groups straddling ranks: sample-level shard_dataset,       */
/* workload.cpp:183-198, with the group unit sample_id / group_size on      */
/* GLOBAL ids, workload.cpp:158-160).  The local batch holds global samples  */
/* [first_sample_id, first_sample_id + n); its first / last local group may  */
/* be partial.  Each rank writes its 6-word boundary record                  */
/* (yatt_filter_boundary_record: {group, first reward bits, any-differs} of  */
/* its first and last local group), the records of all ranks are gathered    */
/* in rank order (world x 6 int64; yatt_peer_allgather_i64 or                */
/* yatt_comm_allgather_i64) and passed as d_all_records: every rank holding  */
/* a piece of a group takes the same exact keep decision.  keep has          */
/* yatt_grpo_num_local_groups(n, first_sample_id, group_size) entries;       */
/* counts[2] counts the groups whose first sample is local (once globally).  */
int yatt_filter_boundary_record(const float* d_rewards, int64_t n_samples,
                                uint64_t first_sample_id, int32_t group_size,
                                int64_t* d_record /* [6] */, void* stream);
int yatt_filter_compact_sharded(const float* d_rewards, const int64_t* d_seq_lens,
                                int64_t n_samples, uint64_t first_sample_id,
                                int32_t group_size, const int64_t* d_all_records,
                                int32_t world, uint8_t* d_keep_groups,
                                int32_t* d_index_map, int64_t* d_new_cu,
                                int64_t* d_counts, void* d_workspace,
                                size_t workspace_bytes, void* stream);
/* Gather variable-length per-token payload of the kept samples:             */
/*   dst[off + new_cu[j] + k] = src[old_cu[map[j]] + k], k < len(map[j])     */
/* for j < *d_n_kept (device count; max_kept bounds the grid).  off =        */
/* *d_dst_offset or 0.  elem_bytes in {1,2,4,8}; old_cu has n_samples+1.     */
int yatt_gather_varlen(const void* d_src, const int64_t* d_old_cu,
                       const int32_t* d_index_map, const int64_t* d_new_cu,
                       const int64_t* d_n_kept, int64_t max_kept,
                       const int64_t* d_dst_offset, int32_t elem_bytes,
                       void* d_dst, void* stream);
/* The same for up to YATT_GATHER_MAX_ARRAYS per-token arrays in ONE launch */
/* (e.g. the 17 B/token payload: token i32, logp/ref_logp/adv f32, mask u8):  */
/* h_srcs / h_dsts / h_elem_bytes are HOST arrays of n_arrays device         */
/* pointers and element sizes; each sample's index lookup is shared.        */
#define YATT_GATHER_MAX_ARRAYS 8
int yatt_gather_varlen_multi(int32_t n_arrays, const void* const* h_srcs,
                             void* const* h_dsts, const int32_t* h_elem_bytes,
                             const int64_t* d_old_cu, const int32_t* d_index_map,
                             const int64_t* d_new_cu, const int64_t* d_n_kept,
                             int64_t max_kept, const int64_t* d_dst_offset,
                             void* stream);
/* Gather fixed-width per-sample rows (metadata, multimodal payload refs):   */
/*   dst[(off + j)*row_bytes ..] = src[map[j]*row_bytes ..], j < *d_n_kept   */
int yatt_gather_rows(const void* d_src, const int32_t* d_index_map,
                     const int64_t* d_n_kept, int64_t max_kept,
                     int64_t row_bytes, const int64_t* d_dst_offset,
                     void* d_dst, void* stream);
/* Microbatch aggregates (simcore.cpp:17-39) over an ordered sample list:   */
/* consecutive chunks of microbatch_size over (prompt_len[i], out_len[i]),  */
/* i < (d_n ? *d_n : n); writes ceil(count/microbatch_size) entries.        */
int yatt_microbatch_aggregates(const int32_t* d_prompt_len,
                               const int32_t* d_out_len, const int64_t* d_n,
                               int64_t n, int32_t microbatch_size,
                               int32_t controller_rank, yatt_mb_agg* d_mbs,
                               void* stream);
/* *d_out = sum_{r < rank} d_counts[r*stride + field] (device, one thread):  */
/* turns all-gathered per-rank counts into this rank's global offset.        */
int yatt_exclusive_offset(const int64_t* d_counts, int32_t nranks, int32_t rank,
                          int32_t stride, int32_t field, int64_t* d_out,
                          void* stream);

/* ------------------------------------------------------------------------ */
/* R10  sort_and_bucket ordering  (replaces balancer.cpp:16-36)              */
/* d_order = indices sorted by length descending, ties by index ascending.   */
/* Bucket cutting + std::shuffle of bucket order stay on the host (the C++   */
/* wrapper yatt::balancer::sort_and_bucket), bit-exact with libstdc++.       */
/* ------------------------------------------------------------------------ */
size_t yatt_sort_order_workspace_bytes(int64_t n);
int yatt_sort_order_desc(const int32_t* d_lengths, int64_t n,
                         uint32_t* d_order, void* d_workspace,
                         size_t workspace_bytes, void* stream);
/* Host helper: full sort_and_bucket through the device sort.  Writes the   */
/* shuffled flat bucket list to h_flat (n entries) and bucket start offsets */
/* to h_bucket_offsets (n_buckets+1 entries, n_buckets = ceil(n/B)).        */
int yatt_sort_and_bucket_host(const int32_t* h_lengths, int64_t n,
                              int32_t batch_size, uint64_t seed,
                              uint32_t* h_flat, int64_t* h_bucket_offsets);

/* ------------------------------------------------------------------------ */
/* Cross-rank collectives (NCCL over NVLink/NVSwitch)                        */
/* ------------------------------------------------------------------------ */
#define YATT_COMM_ID_BYTES 128
typedef struct yatt_comm* yatt_comm_t;
int yatt_comm_unique_id(uint8_t* h_id /* YATT_COMM_ID_BYTES */);
int yatt_comm_init(int32_t nranks, int32_t rank, const uint8_t* h_id,
                   yatt_comm_t* out_comm);
int yatt_comm_destroy(yatt_comm_t comm);
int yatt_comm_allreduce_f64(yatt_comm_t comm, double* d_buf, int64_t count,
                            void* stream);
int yatt_comm_allreduce_i64(yatt_comm_t comm, int64_t* d_buf, int64_t count,
                            void* stream);
int yatt_comm_allgather_i64(yatt_comm_t comm, const int64_t* d_send,
                            int64_t* d_recv, int64_t count_per_rank,
                            void* stream);

/* ------------------------------------------------------------------------ */
/* Synthetic inputs (bench / parity support; same recipe in oracle/)         */
/* ------------------------------------------------------------------------ */
/* Logits for global rows [row0, row0+rows): see DESIGN.md "Synthetic data". */
int yatt_synth_logits(uint64_t seed, int64_t row0, int64_t rows, int32_t vocab,
                      uint16_t* d_policy, uint16_t* d_ref, int32_t* d_targets,
                      void* stream);
/* out[i] = f(kind, uniform/int draw of hash_key({seed, stream_id, i0+i})).  */
enum yatt_synth_kind {
  YATT_SYNTH_LOGP = 0,      /* -k/64, k in [0,1023]                          */
  YATT_SYNTH_OLD_DELTA = 1, /* k/256, k in [-64,63]  (added to a base)       */
  YATT_SYNTH_ADV = 2,       /* k/64,  k in [-128,127]                        */
  YATT_SYNTH_KL = 3,        /* k/1024, k in [0,255]                          */
  YATT_SYNTH_VALUE = 4,     /* k/1024, k in [-1024,1023]                     */
  YATT_SYNTH_REWARD = 5     /* binary group rewards           */
};
int yatt_synth_floats(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n,
                      int32_t kind, int32_t group_size, const float* d_base,
                      float* d_out, void* stream);

/* ------------------------------------------------------------------------ */
/* Peer-memory group (one node): compute + all-reduce in ONE kernel over     */
/* NVLink.  Each rank creates its group member (a small device buffer with   */
/* a CUDA IPC handle), exchanges the handles out of band (torch.distributed  */
/* all_gather / the controller rendezvous), then connects.  Calls are        */
/* collective (every rank, same order); results are bit-identical on every   */
/* rank (rank-ordered sum).  A peer that never arrives makes the call write  */
/* NaN (-1 for the int64 calls) after 10 s of wall time and sets             */
/* yatt_peer_status to 1 instead of hanging; destroy the group after that.   */
/* ------------------------------------------------------------------------ */
#define YATT_PEER_MAX_WORLD 8
#define YATT_PEER_HANDLE_BYTES 64
typedef struct yatt_peer* yatt_peer_t;
int yatt_peer_create(int32_t world, int32_t rank, yatt_peer_t* out_peer,
                     uint8_t* h_handle /* YATT_PEER_HANDLE_BYTES */);
int yatt_peer_connect(yatt_peer_t peer,
                      const uint8_t* h_handles /* world * YATT_PEER_HANDLE_BYTES */);
int yatt_peer_destroy(yatt_peer_t peer);
int yatt_peer_status(yatt_peer_t peer, int32_t* h_status);
/* d_out[i] = sum over ranks of d_in[i], i < n <= 16. */
int yatt_peer_allreduce_f64(yatt_peer_t peer, const double* d_in, int32_t n,
                            double* d_out, void* stream);
/* All-gather + exclusive scan over ranks of n <= 16 int64 counters in one    */
/* kernel: d_prefix[i] = sum over lower ranks, d_total[i] = sum over all      */
/* (either may be NULL) — e.g. the dynamic-sampling counts -> this rank's     */
/* offset into the global packed layout (yatt_gather_* d_dst_offset).         */
int yatt_peer_scan_i64(yatt_peer_t peer, const int64_t* d_in, int32_t n,
                       int64_t* d_prefix, int64_t* d_total, void* stream);
/* All-gather of n <= YATT_PEER_GATHER_MAX_WORDS int64 words per rank:       */
/* d_out[world * n], rank-major, identical on all ranks (the dynamic-        */
/* sampling round reports + microbatch aggregates; -1 everywhere on a peer   */
/* timeout).  Collective, same call order on every rank.                     */
#define YATT_PEER_GATHER_MAX_WORDS 16384
int yatt_peer_allgather_i64(yatt_peer_t peer, const int64_t* d_in, int32_t n,
                            int64_t* d_out, void* stream);

/* Group-level ops of a rank whose shard may split groups with its           */
/* neighbours, in one call over the peer group: boundary record -> peer      */
/* all-gather -> device merge -> the op (all stream-ordered; collective:     */
/* every rank calls).  Advantages equal a single rank's to fp64 rounding of  */
/* the merged moments; the filter's layout is bit-exact.  Workspace:         */
/* yatt_straddle_workspace_bytes(n_samples, first_sample_id, G, world).      */
size_t yatt_straddle_workspace_bytes(int64_t n_samples, uint64_t first_sample_id,
                                     int32_t group_size, int32_t world);
int yatt_peer_world(yatt_peer_t p, int32_t* h_world, int32_t* h_rank);

/* The multi-rank dynamic-sampling step with ONE exchange (replaces the      */
/* per-round submit_round / feed_round / continue protocol, demo.cpp:468-476 */
/* and simcore.cpp:470-490): this rank's controller shard (n samples staged  */
/* with yatt_rounds_stage(h, n, 1, ...)) runs every round in one persistent  */
/* kernel, then every rank's reports + microbatch aggregates are all-gathered */
/* over the peer group.  Afterwards yatt_rounds_result(h) is the GLOBAL view: */
/* reports[round][rank] (rounds = max over ranks; a finished shard reports    */
/* zeros) and the microbatches in that order; the staged outputs are this     */
/* rank's samples.  Collective: every rank calls, same step and params.      */
int yatt_peer_rounds_run(yatt_peer_t peer, yatt_rounds_t h, int64_t n, int32_t step_index,
                         const yatt_round_params* params, int32_t want_first_lens,
                         void* stream);
int yatt_peer_grpo_advantages(yatt_peer_t p, const float* d_rewards, int64_t n_samples,
                              uint64_t first_sample_id, int32_t group_size, float eps,
                              int32_t norm_by_std, float* d_sample_adv, void* d_workspace,
                              size_t workspace_bytes, void* stream);
int yatt_peer_filter_compact(yatt_peer_t p, const float* d_rewards,
                             const int64_t* d_seq_lens, int64_t n_samples,
                             uint64_t first_sample_id, int32_t group_size,
                             uint8_t* d_keep_groups, int32_t* d_index_map,
                             int64_t* d_new_cu, int64_t* d_counts, void* d_workspace,
                             size_t workspace_bytes, void* stream);
/* yatt_policy_loss whose final reduction also all-reduces across the group:  */
/* d_sums holds the GLOBAL sums on every rank (one kernel after the partials). */
int yatt_policy_loss_allreduce(yatt_peer_t peer, const float* d_logp,
                               const float* d_old_logp, const float* d_advantages,
                               const float* d_kl, const float* d_entropy,
                               const uint8_t* d_mask, int64_t n_tokens,
                               const int64_t* d_cu_seqlens, int64_t n_seqs,
                               const yatt_loss_config* config,
                               yatt_loss_sums* d_sums, void* d_workspace,
                               size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* YATT_CUDA_H_ */
