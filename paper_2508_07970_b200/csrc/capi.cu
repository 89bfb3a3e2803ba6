// capi.cu — extern "C" entry points of include/yatt_cuda.h.
//
// Thin: validates, converts void* streams, forwards to the *_launch functions
// of the kernel files, and keeps a thread-local last-error message.  The host
// buffer variants (yatt_token_stats_host, yatt_sort_and_bucket_host) own the
// H2D/D2H copies — they are what a C++ caller holding STL/host data uses, and
// what bench.py times as the end-to-end path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <random>
#include <vector>

#include "common.cuh"

namespace yattb {

// ---- kernel-file entry points -------------------------------------------
int token_stats_launch(const uint16_t*, const uint16_t*, const int32_t*, const uint8_t*, int64_t,
                       int32_t, int32_t, float*, float*, float*, float*, cudaStream_t);
int synth_logits_launch(uint64_t, int64_t, int64_t, int32_t, uint16_t*, uint16_t*, int32_t*,
                        cudaStream_t);
int synth_floats_launch(uint64_t, uint64_t, int64_t, int64_t, int32_t, int32_t, const float*,
                        float*, cudaStream_t);
int64_t grpo_num_local_groups(int64_t, uint64_t, int32_t);
int grpo_moments_launch(const float*, int64_t, uint64_t, int32_t, double*, cudaStream_t);
int grpo_adv_launch(const float*, int64_t, uint64_t, int32_t, float, int32_t, const double*,
                    float*, cudaStream_t);
int broadcast_launch(const float*, const int64_t*, int64_t, const uint8_t*, float*, cudaStream_t);
int gae_launch(const float*, const float*, const uint8_t*, const int64_t*, int64_t, int64_t, float,
               float, float*, float*, void*, size_t, cudaStream_t, double* moments = nullptr);
size_t gae_workspace_bytes(int64_t);
size_t moments_workspace_bytes();
int masked_moments_launch(const float*, const uint8_t*, int64_t, double*, double*, cudaStream_t);
int whiten_launch(float*, const uint8_t*, int64_t, const double*, int32_t, cudaStream_t);
size_t loss_workspace_bytes();
int policy_loss_launch(const float*, const float*, const float*, const float*, const float*,
                       const uint8_t*, int64_t, const int64_t*, int64_t, const yatt_loss_config*,
                       yatt_loss_sums*, void*, size_t, cudaStream_t);
double loss_finalize(const yatt_loss_sums*, const yatt_loss_config*);
size_t compact_workspace_bytes(int64_t);
int filter_compact_launch(const float*, const int64_t*, int64_t, uint64_t, int32_t, const int64_t*,
                          int32_t, uint8_t*, int32_t*,
                          int64_t*, int64_t*, void*, size_t, cudaStream_t);
int gather_varlen_multi_launch(int32_t, const void* const*, void* const*, const int32_t*,
                               const int64_t*, const int32_t*, const int64_t*, const int64_t*,
                               int64_t, const int64_t*, cudaStream_t);
int gather_varlen_launch(const void*, const int64_t*, const int32_t*, const int64_t*,
                         const int64_t*, int64_t, const int64_t*, int32_t, void*, cudaStream_t);
int gather_rows_launch(const void*, const int32_t*, const int64_t*, int64_t, int64_t,
                       const int64_t*, void*, cudaStream_t);
int microbatch_launch(const int32_t*, const int32_t*, const int64_t*, int64_t, int32_t, int32_t,
                      yatt_mb_agg*, cudaStream_t);
int exclusive_offset_launch(const int64_t*, int32_t, int32_t, int32_t, int32_t, int64_t*,
                            cudaStream_t);
int validate_dist(const yatt_length_dist*);
int validate_rejection(const yatt_rejection_config*);
int lengths_launch(const yatt_length_dist*, uint64_t, uint64_t, uint64_t, uint64_t,
                   const uint64_t*, int64_t, int32_t*, cudaStream_t);
int lengths_host(const yatt_length_dist*, uint64_t, uint64_t, uint64_t, uint64_t, const uint64_t*,
                 int64_t, int32_t*);
int uncertified_draws(int64_t*, int32_t);
int rejection_launch(const yatt_sample*, int64_t, int32_t, int32_t, const yatt_rejection_config*,
                     uint64_t, uint8_t*, cudaStream_t);
int shard_round_launch(yatt_sample*, const int64_t*, int32_t, int32_t, int32_t, int32_t,
                       const yatt_round_params*, yatt_round_report*, yatt_mb_agg*, cudaStream_t);
size_t sort_workspace_bytes(int64_t);
int sort_order_launch(const int32_t*, int64_t, uint32_t*, void*, size_t, cudaStream_t);
int reduce_reports_launch(const yatt_round_report*, int32_t, int64_t*, cudaStream_t);
size_t lmhead_workspace_bytes(int64_t, int32_t, int32_t);
int lmhead_token_stats_launch(const uint16_t*, const uint16_t*, const int32_t*, int64_t, int32_t,
                              int32_t, int32_t, float*, float*, float*, void*, size_t,
                              cudaStream_t);
int kl_from_logps_launch(const float*, const float*, int64_t, int32_t, float*, cudaStream_t);
int grad_coef_launch(const uint16_t*, const uint16_t*, const int32_t*, const float*, const float*,
                     const float*, const float*, const float*, const float*, const uint8_t*,
                     int64_t, int32_t, const int64_t*, int64_t, const yatt_loss_config*, int32_t,
                     double, float*, cudaStream_t);
int policy_loss_grad_launch(const uint16_t*, const uint16_t*, const int32_t*, const uint8_t*,
                            const float*,
                            const float*, const float*, int64_t, int32_t, const int64_t*, int64_t,
                            const yatt_loss_config*, int32_t, double, float*, float*, float*,
                            uint16_t*, void*, size_t, cudaStream_t);
size_t policy_loss_grad_workspace_bytes(int64_t, int32_t);
int logits_backward_launch(const uint16_t*, const uint16_t*, const int32_t*, const uint8_t*,
                           int64_t, int32_t, const float*, int32_t, uint16_t*, cudaStream_t);

// ---- errors ---------------------------------------------------------------
namespace {
thread_local char g_err[1024] = "";
}

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(YATT_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return YATT_OK;
}

int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

int ensure_dynamic_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  YATT_TRY_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == kernel && d.second == dev) return YATT_OK;
  YATT_TRY_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.emplace_back(kernel, dev);
  return YATT_OK;
}

// Grow-only device buffer cache for the host-buffer entry points.
namespace {
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int reserve(size_t need) {
    if (need <= bytes) return YATT_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    YATT_TRY_CUDA(cudaMalloc(&p, need));
    bytes = need;
    return YATT_OK;
  }
};
}  // namespace

}  // namespace yattb

using namespace yattb;

// Natural-alignment contract of every pointer argument (the kernels issue
// vector / 64-bit accesses): a misaligned pointer is a YATT_ERR_CONFIG, not a
// device fault that poisons the context.  Null pointers pass (optional args).
#define YATT_ALIGNED(fn, ptr, a)                                                          \
  YATT_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & uintptr_t((a) - 1)) == 0, YATT_ERR_CONFIG, \
               "%s: %s must be %d-byte aligned", fn, #ptr, int(a))
#define YATT_ALIGNED4(fn, a, b, c, d) \
  do {                                \
    YATT_ALIGNED(fn, a, 4);           \
    YATT_ALIGNED(fn, b, 4);           \
    YATT_ALIGNED(fn, c, 4);           \
    YATT_ALIGNED(fn, d, 4);           \
  } while (0)

extern "C" {

const char* yatt_last_error_message(void) { return yattb::g_err; }
int yatt_abi_version(void) { return 3; }

int yatt_device_info(int device, char* name, int name_len, int* sm_major, int* sm_minor,
                     int* nsms) {
  cudaDeviceProp prop;
  YATT_TRY_CUDA(cudaGetDeviceProperties(&prop, device));
  if (name && name_len > 0) {
    std::strncpy(name, prop.name, size_t(name_len) - 1);
    name[name_len - 1] = 0;
  }
  if (sm_major) *sm_major = prop.major;
  if (sm_minor) *sm_minor = prop.minor;
  if (nsms) *nsms = prop.multiProcessorCount;
  return YATT_OK;
}

int yatt_shard_dataset(uint64_t total, int32_t p, int32_t r, uint64_t* begin, uint64_t* end) {
  YATT_REQUIRE(p > 0, YATT_ERR_CONFIG, "num_controllers must be positive");
  YATT_REQUIRE(r >= 0 && r < p, YATT_ERR_RANK, "controller_rank out of range");
  const uint64_t P = uint64_t(p), R = uint64_t(r);
  const uint64_t base = total / P, rem = total % P;
  const uint64_t b = R * base + (R < rem ? R : rem);
  if (begin) *begin = b;
  if (end) *end = b + base + (R < rem ? 1 : 0);
  return YATT_OK;
}

int yatt_sample_lengths_keyed(const yatt_length_dist* d, uint64_t seed, uint64_t stream_id,
                              uint64_t step, uint64_t round, const uint64_t* ids, int64_t n,
                              int32_t* out, void* stream) {
  YATT_ALIGNED("sample_lengths_keyed", ids, 8);
  YATT_ALIGNED("sample_lengths_keyed", out, 4);
  return lengths_launch(d, seed, stream_id, step, round, ids, n, out, as_stream(stream));
}

int yatt_sample_lengths_host(const yatt_length_dist* d, uint64_t seed, uint64_t stream_id,
                             uint64_t step, uint64_t round, const uint64_t* h_ids, int64_t n,
                             int32_t* h_out) {
  return lengths_host(d, seed, stream_id, step, round, h_ids, n, h_out);
}

int yatt_uncertified_draws(int64_t* h_count, int32_t reset) {
  return uncertified_draws(h_count, reset);
}

int yatt_rejection_flags(const yatt_sample* s, int64_t n, int32_t step, int32_t round,
                         const yatt_rejection_config* c, uint64_t seed, uint8_t* out,
                         void* stream) {
  YATT_ALIGNED("rejection_flags", s, 8);
  return rejection_launch(s, n, step, round, c, seed, out, as_stream(stream));
}

int yatt_shard_round(yatt_sample* samples, const int64_t* h_off, int32_t nshards,
                     int32_t first_rank, int32_t step, int32_t round, const yatt_round_params* p,
                     yatt_round_report* reports, yatt_mb_agg* mbs, void* stream) {
  YATT_ALIGNED("shard_round", samples, 8);
  YATT_ALIGNED("shard_round", reports, 8);
  YATT_ALIGNED("shard_round", mbs, 8);
  return shard_round_launch(samples, h_off, nshards, first_rank, step, round, p, reports, mbs,
                            as_stream(stream));
}

size_t yatt_lmhead_workspace_bytes(int64_t rows, int32_t vocab, int32_t n_split) {
  return lmhead_workspace_bytes(rows, vocab, n_split);
}

int yatt_lmhead_token_stats(const uint16_t* hidden, const uint16_t* w, const int32_t* tgt,
                            int64_t rows, int32_t d, int32_t vocab, int32_t n_split, float* logp,
                            float* ent, float* lse, void* ws, size_t ws_bytes, void* stream) {
  YATT_ALIGNED4("lmhead_token_stats", tgt, logp, ent, lse);
  YATT_ALIGNED("lmhead_token_stats", ws, 16);
  return lmhead_token_stats_launch(hidden, w, tgt, rows, d, vocab, n_split, logp, ent, lse, ws,
                                   ws_bytes, as_stream(stream));
}

int yatt_kl_from_logps(const float* logp, const float* ref_logp, int64_t n, int32_t mode,
                       float* kl, void* stream) {
  YATT_ALIGNED4("kl_from_logps", logp, ref_logp, kl, nullptr);
  return kl_from_logps_launch(logp, ref_logp, n, mode, kl, as_stream(stream));
}

int yatt_reduce_round_reports(const yatt_round_report* r, int32_t n, int64_t* out, void* stream) {
  YATT_ALIGNED("reduce_round_reports", r, 8);
  YATT_ALIGNED("reduce_round_reports", out, 8);
  return reduce_reports_launch(r, n, out, as_stream(stream));
}

int yatt_token_stats(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                     const uint8_t* mask, int64_t rows, int32_t vocab, int32_t kl_mode,
                     float* logp, float* ref_logp, float* ent, float* kl, void* stream) {
  YATT_ALIGNED4("token_stats", logp, ref_logp, ent, kl);
  YATT_ALIGNED("token_stats", tgt, 4);
  YATT_ALIGNED("token_stats", pol, 2);
  YATT_ALIGNED("token_stats", ref, 2);
  return token_stats_launch(pol, ref, tgt, mask, rows, vocab, kl_mode, logp, ref_logp, ent, kl,
                            as_stream(stream));
}

int yatt_token_stats_host(const uint16_t* h_pol, const uint16_t* h_ref, const int32_t* h_tgt,
                          const uint8_t* h_mask, int64_t rows, int32_t vocab, int32_t kl_mode,
                          float* h_logp, float* h_ref_logp, float* h_ent, float* h_kl) {
  YATT_REQUIRE(vocab > 0, YATT_ERR_CONFIG, "token_stats: vocab must be positive (got %d)", vocab);
  YATT_REQUIRE(rows >= 0, YATT_ERR_CONFIG, "token_stats: rows must be >= 0");
  if (rows == 0) return YATT_OK;
  YATT_REQUIRE(h_logp != nullptr, YATT_ERR_CONFIG, "token_stats: logp output is required");
  YATT_REQUIRE(h_pol && h_ref && h_tgt, YATT_ERR_CONFIG, "token_stats: null input pointer");
  // ~128 MiB per tensor per chunk: long enough to amortise per-copy
  // overhead, short enough that two slots overlap copy and compute.
  const int64_t row_bytes = int64_t(vocab) * 2;
  const int64_t chunk = max64(1, min64(rows, (int64_t(128) << 20) / row_bytes));
  struct Slot {
    DevBuf pol, ref, tgt, mask, out;
    cudaStream_t st = nullptr;
  };
  static thread_local Slot slots[2];
  for (Slot& s : slots) {
    if (!s.st) YATT_TRY_CUDA(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    int rc = s.pol.reserve(size_t(chunk * row_bytes));
    if (!rc) rc = s.ref.reserve(size_t(chunk * row_bytes));
    if (!rc) rc = s.tgt.reserve(size_t(chunk) * 4);
    if (!rc) rc = s.mask.reserve(size_t(chunk));
    if (!rc) rc = s.out.reserve(size_t(chunk) * 16);
    if (rc) return rc;
  }
  int k = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk, k ^= 1) {
    Slot& s = slots[k];
    const int64_t n = std::min(chunk, rows - r0);
    float* o = static_cast<float*>(s.out.p);
    YATT_TRY_CUDA(cudaMemcpyAsync(s.pol.p, h_pol + r0 * vocab, size_t(n * row_bytes),
                                  cudaMemcpyHostToDevice, s.st));
    YATT_TRY_CUDA(cudaMemcpyAsync(s.ref.p, h_ref + r0 * vocab, size_t(n * row_bytes),
                                  cudaMemcpyHostToDevice, s.st));
    YATT_TRY_CUDA(cudaMemcpyAsync(s.tgt.p, h_tgt + r0, size_t(n) * 4, cudaMemcpyHostToDevice, s.st));
    if (h_mask)
      YATT_TRY_CUDA(cudaMemcpyAsync(s.mask.p, h_mask + r0, size_t(n), cudaMemcpyHostToDevice, s.st));
    int rc = token_stats_launch(static_cast<uint16_t*>(s.pol.p), static_cast<uint16_t*>(s.ref.p),
                                static_cast<int32_t*>(s.tgt.p),
                                h_mask ? static_cast<uint8_t*>(s.mask.p) : nullptr, n, vocab,
                                kl_mode, o, o + chunk, o + 2 * chunk, o + 3 * chunk, s.st);
    if (rc) return rc;
    float* dst[4] = {h_logp, h_ref_logp, h_ent, h_kl};
    for (int f = 0; f < 4; ++f)
      if (dst[f])
        YATT_TRY_CUDA(cudaMemcpyAsync(dst[f] + r0, o + f * chunk, size_t(n) * 4,
                                      cudaMemcpyDeviceToHost, s.st));
  }
  for (Slot& s : slots) YATT_TRY_CUDA(cudaStreamSynchronize(s.st));
  return YATT_OK;
}

int yatt_grpo_step_host(const uint16_t* h_pol, const uint16_t* h_ref, const int32_t* h_tgt,
                        const uint8_t* h_mask, int64_t rows, int32_t vocab,
                        const float* h_rewards, int64_t n_samples, uint64_t first_id, int32_t G,
                        const float* h_old, const yatt_loss_config* cfg, int32_t kl_mode,
                        yatt_loss_sums* h_sums, float* h_stats) {
  YATT_REQUIRE(vocab > 0 && rows > 0 && n_samples > 0 && rows % n_samples == 0, YATT_ERR_CONFIG,
               "grpo_step: rows must be a positive multiple of n_samples");
  YATT_REQUIRE(h_pol && h_ref && h_tgt && h_rewards && h_old && cfg && h_sums, YATT_ERR_CONFIG,
               "grpo_step: null argument");
  const int64_t T = rows / n_samples;
  const int64_t row_bytes = int64_t(vocab) * 2;
  const int64_t chunk = max64(1, min64(rows, (int64_t(128) << 20) / row_bytes));
  struct Slot {
    DevBuf pol, ref, tgt;
    cudaStream_t st = nullptr;
  };
  static thread_local Slot slots[2];
  static thread_local DevBuf stats, mask, rew, adv, tadv, old, cu, sums, ws;
  for (Slot& s : slots) {
    if (!s.st) YATT_TRY_CUDA(cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
    int rc = s.pol.reserve(size_t(chunk * row_bytes));
    if (!rc) rc = s.ref.reserve(size_t(chunk * row_bytes));
    if (!rc) rc = s.tgt.reserve(size_t(chunk) * 4);
    if (rc) return rc;
  }
  int rc = stats.reserve(size_t(rows) * 16);
  if (!rc) rc = mask.reserve(size_t(rows));
  if (!rc) rc = rew.reserve(size_t(n_samples) * 4);
  if (!rc) rc = adv.reserve(size_t(n_samples) * 4);
  if (!rc) rc = tadv.reserve(size_t(rows) * 4);
  if (!rc) rc = old.reserve(size_t(rows) * 4);
  if (!rc) rc = cu.reserve(size_t(n_samples + 1) * 8);
  if (!rc) rc = sums.reserve(sizeof(yatt_loss_sums));
  if (!rc) rc = ws.reserve(loss_workspace_bytes());
  if (rc) return rc;
  float* st4 = static_cast<float*>(stats.p);
  uint8_t* dmask = static_cast<uint8_t*>(mask.p);
  // 1. stream the logits through two staging slots, A1 into the stats arrays
  int k = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk, k ^= 1) {
    Slot& s = slots[k];
    const int64_t n = min64(chunk, rows - r0);
    YATT_TRY_CUDA(cudaMemcpyAsync(s.pol.p, h_pol + r0 * vocab, size_t(n * row_bytes),
                                  cudaMemcpyHostToDevice, s.st));
    YATT_TRY_CUDA(cudaMemcpyAsync(s.ref.p, h_ref + r0 * vocab, size_t(n * row_bytes),
                                  cudaMemcpyHostToDevice, s.st));
    YATT_TRY_CUDA(cudaMemcpyAsync(s.tgt.p, h_tgt + r0, size_t(n) * 4, cudaMemcpyHostToDevice, s.st));
    if (h_mask)
      YATT_TRY_CUDA(cudaMemcpyAsync(dmask + r0, h_mask + r0, size_t(n), cudaMemcpyHostToDevice,
                                    s.st));
    else
      YATT_TRY_CUDA(cudaMemsetAsync(dmask + r0, 1, size_t(n), s.st));
    rc = token_stats_launch(static_cast<uint16_t*>(s.pol.p), static_cast<uint16_t*>(s.ref.p),
                            static_cast<int32_t*>(s.tgt.p), dmask + r0, n, vocab, kl_mode,
                            st4 + r0, st4 + rows + r0, st4 + 2 * rows + r0, st4 + 3 * rows + r0,
                            s.st);
    if (rc) return rc;
  }
  YATT_TRY_CUDA(cudaStreamSynchronize(slots[1].st));
  cudaStream_t st = slots[0].st;
  // 2. GRPO advantages -> tokens -> loss sums
  std::vector<int64_t> hcu(static_cast<size_t>(n_samples + 1));
  for (int64_t i = 0; i <= n_samples; ++i) hcu[size_t(i)] = i * T;
  YATT_TRY_CUDA(cudaMemcpyAsync(rew.p, h_rewards, size_t(n_samples) * 4, cudaMemcpyHostToDevice, st));
  YATT_TRY_CUDA(cudaMemcpyAsync(old.p, h_old, size_t(rows) * 4, cudaMemcpyHostToDevice, st));
  YATT_TRY_CUDA(cudaMemcpyAsync(cu.p, hcu.data(), hcu.size() * 8, cudaMemcpyHostToDevice, st));
  rc = grpo_adv_launch(static_cast<float*>(rew.p), n_samples, first_id, G, 1e-6f, 1, nullptr,
                       static_cast<float*>(adv.p), st);
  if (!rc)
    rc = broadcast_launch(static_cast<float*>(adv.p), static_cast<int64_t*>(cu.p), n_samples, dmask,
                          static_cast<float*>(tadv.p), st);
  if (!rc)
    rc = policy_loss_launch(st4, static_cast<float*>(old.p), static_cast<float*>(tadv.p),
                            st4 + 3 * rows, st4 + 2 * rows, dmask, rows,
                            static_cast<int64_t*>(cu.p), n_samples, cfg,
                            static_cast<yatt_loss_sums*>(sums.p), ws.p, ws.bytes, st);
  if (rc) return rc;
  YATT_TRY_CUDA(cudaMemcpyAsync(h_sums, sums.p, sizeof(yatt_loss_sums), cudaMemcpyDeviceToHost, st));
  if (h_stats)
    YATT_TRY_CUDA(cudaMemcpyAsync(h_stats, st4, size_t(rows) * 16, cudaMemcpyDeviceToHost, st));
  YATT_TRY_CUDA(cudaStreamSynchronize(st));
  return YATT_OK;
}

int64_t yatt_grpo_num_local_groups(int64_t n, uint64_t first_id, int32_t G) {
  return grpo_num_local_groups(n, first_id, G);
}

int yatt_grpo_group_moments(const float* r, int64_t n, uint64_t first_id, int32_t G, double* out,
                            void* stream) {
  YATT_ALIGNED("grpo_group_moments", r, 4);
  YATT_ALIGNED("grpo_group_moments", out, 8);
  return grpo_moments_launch(r, n, first_id, G, out, as_stream(stream));
}

int yatt_grpo_advantages(const float* r, int64_t n, uint64_t first_id, int32_t G, float eps,
                         int32_t norm_by_std, const double* moments, float* adv, void* stream) {
  YATT_ALIGNED4("grpo_advantages", r, adv, nullptr, nullptr);
  YATT_ALIGNED("grpo_advantages", moments, 8);
  return grpo_adv_launch(r, n, first_id, G, eps, norm_by_std, moments, adv, as_stream(stream));
}

int yatt_broadcast_to_tokens(const float* vals, const int64_t* cu, int64_t nsamples,
                             const uint8_t* mask, float* out, int64_t n_tokens, void* stream) {
  YATT_ALIGNED4("broadcast_to_tokens", vals, out, nullptr, nullptr);
  YATT_ALIGNED("broadcast_to_tokens", cu, 8);
  (void)n_tokens;
  return broadcast_launch(vals, cu, nsamples, mask, out, as_stream(stream));
}

size_t yatt_gae_workspace_bytes(int64_t n_tokens) { return gae_workspace_bytes(n_tokens); }

int yatt_gae(const float* values, const float* rewards, const uint8_t* mask, const int64_t* cu,
             int64_t nseq, int64_t n_tokens, float gamma, float lam, float* adv, float* ret,
             void* ws, size_t ws_bytes, void* stream) {
  YATT_ALIGNED4("gae", values, rewards, adv, ret);
  YATT_ALIGNED("gae", cu, 8);
  YATT_ALIGNED("gae", ws, 16);
  return gae_launch(values, rewards, mask, cu, nseq, n_tokens, gamma, lam, adv, ret, ws, ws_bytes,
                    as_stream(stream));
}

int yatt_gae_with_moments(const float* values, const float* rewards, const uint8_t* mask,
                          const int64_t* cu, int64_t nseq, int64_t n_tokens, float gamma,
                          float lam, float* adv, float* ret, double* moments, void* ws,
                          size_t ws_bytes, void* stream) {
  YATT_ALIGNED4("gae_with_moments", values, rewards, adv, ret);
  YATT_ALIGNED("gae_with_moments", cu, 8);
  YATT_ALIGNED("gae_with_moments", ws, 16);
  YATT_ALIGNED("gae_with_moments", moments, 8);
  YATT_REQUIRE(moments != nullptr, YATT_ERR_CONFIG, "gae_with_moments: null moments");
  return gae_launch(values, rewards, mask, cu, nseq, n_tokens, gamma, lam, adv, ret, ws, ws_bytes,
                    as_stream(stream), moments);
}

size_t yatt_masked_moments_workspace_bytes(void) { return moments_workspace_bytes(); }

int yatt_masked_moments(const float* x, const uint8_t* mask, int64_t n, double* out, void* ws,
                        size_t ws_bytes, void* stream) {
  YATT_ALIGNED("masked_moments", x, 4);
  YATT_ALIGNED("masked_moments", out, 8);
  YATT_ALIGNED("masked_moments", ws, 8);
  YATT_REQUIRE(ws != nullptr && ws_bytes >= moments_workspace_bytes(), YATT_ERR_WORKSPACE,
               "masked_moments: workspace too small");
  return masked_moments_launch(x, mask, n, out, static_cast<double*>(ws), as_stream(stream));
}

int yatt_whiten(float* x, const uint8_t* mask, int64_t n, const double* mom, int32_t shift,
                void* stream) {
  YATT_ALIGNED("whiten", x, 4);
  YATT_ALIGNED("whiten", mom, 8);
  return whiten_launch(x, mask, n, mom, shift, as_stream(stream));
}

size_t yatt_policy_loss_workspace_bytes(int64_t, int64_t, int32_t) {
  return loss_workspace_bytes();
}

int yatt_policy_loss(const float* logp, const float* old_logp, const float* adv, const float* kl,
                     const float* ent, const uint8_t* mask, int64_t n, const int64_t* cu,
                     int64_t nseq, const yatt_loss_config* cfg, yatt_loss_sums* sums, void* ws,
                     size_t ws_bytes, void* stream) {
  YATT_ALIGNED4("policy_loss", logp, old_logp, adv, kl);
  YATT_ALIGNED("policy_loss", ent, 4);
  YATT_ALIGNED("policy_loss", cu, 8);
  YATT_ALIGNED("policy_loss", sums, 8);
  YATT_ALIGNED("policy_loss", ws, 8);
  return policy_loss_launch(logp, old_logp, adv, kl, ent, mask, n, cu, nseq, cfg, sums, ws,
                            ws_bytes, as_stream(stream));
}

double yatt_loss_finalize(const yatt_loss_sums* s, const yatt_loss_config* c) {
  return loss_finalize(s, c);
}

int yatt_policy_grad_coef(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                          const float* logp, const float* ref_logp, const float* old_logp,
                          const float* adv, const float* ent, const float* kl,
                          const uint8_t* mask, int64_t n, int32_t vocab, const int64_t* cu,
                          int64_t nseq, const yatt_loss_config* cfg, int32_t kl_mode,
                          double norm, float* coef, void* stream) {
  YATT_ALIGNED4("policy_grad_coef", logp, ref_logp, old_logp, adv);
  YATT_ALIGNED4("policy_grad_coef", ent, kl, tgt, nullptr);
  YATT_ALIGNED("policy_grad_coef", cu, 8);
  YATT_ALIGNED("policy_grad_coef", coef, 16);
  return grad_coef_launch(pol, ref, tgt, logp, ref_logp, old_logp, adv, ent, kl, mask, n, vocab,
                          cu, nseq, cfg, kl_mode, norm, coef, as_stream(stream));
}

int yatt_logits_backward(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                         const uint8_t* mask, int64_t rows, int32_t vocab, const float* coef,
                         int32_t full_kl, uint16_t* grad, void* stream) {
  YATT_ALIGNED("logits_backward", tgt, 4);
  YATT_ALIGNED("logits_backward", coef, 16);
  return logits_backward_launch(pol, ref, tgt, mask, rows, vocab, coef, full_kl, grad,
                                as_stream(stream));
}

size_t yatt_policy_loss_grad_workspace_bytes(int64_t rows, int32_t agg_mode) {
  return policy_loss_grad_workspace_bytes(rows, agg_mode);
}

int yatt_policy_loss_grad(const uint16_t* pol, const uint16_t* ref, const int32_t* tgt,
                          const uint8_t* mask,
                          const float* ref_logp, const float* old_logp, const float* adv,
                          int64_t rows, int32_t vocab, const int64_t* cu, int64_t nseq,
                          const yatt_loss_config* cfg, int32_t kl_mode, double norm, float* logp,
                          float* ent, float* kl, uint16_t* grad, void* ws, size_t ws_bytes,
                          void* stream) {
  YATT_ALIGNED("policy_loss_grad", pol, 16);
  YATT_ALIGNED("policy_loss_grad", grad, 16);
  YATT_ALIGNED("policy_loss_grad", ref, 16);
  YATT_ALIGNED4("policy_loss_grad", tgt, ref_logp, old_logp, adv);
  YATT_ALIGNED4("policy_loss_grad", logp, ent, kl, ws);
  YATT_ALIGNED("policy_loss_grad", cu, 8);
  return policy_loss_grad_launch(pol, ref, tgt, mask, ref_logp, old_logp, adv, rows, vocab, cu,
                                 nseq,
                                 cfg, kl_mode, norm, logp, ent, kl, grad, ws, ws_bytes,
                                 as_stream(stream));
}

size_t yatt_filter_compact_workspace_bytes(int64_t n) { return compact_workspace_bytes(n); }

int yatt_filter_compact(const float* r, const int64_t* lens, int64_t n, int32_t G, uint8_t* keep,
                        int32_t* map, int64_t* new_cu, int64_t* counts, void* ws, size_t ws_bytes,
                        void* stream) {
  YATT_ALIGNED4("filter_compact", r, map, nullptr, nullptr);
  YATT_ALIGNED("filter_compact", lens, 8);
  YATT_ALIGNED("filter_compact", new_cu, 8);
  YATT_ALIGNED("filter_compact", counts, 8);
  YATT_ALIGNED("filter_compact", ws, 8);
  return filter_compact_launch(r, lens, n, 0, G, nullptr, 1, keep, map, new_cu, counts, ws,
                               ws_bytes, as_stream(stream));
}

int yatt_filter_compact_sharded(const float* r, const int64_t* lens, int64_t n,
                                uint64_t first_sample_id, int32_t G, const int64_t* d_all_records,
                                int32_t world, uint8_t* keep, int32_t* map, int64_t* new_cu,
                                int64_t* counts, void* ws, size_t ws_bytes, void* stream) {
  YATT_ALIGNED4("filter_compact_sharded", r, map, nullptr, nullptr);
  YATT_ALIGNED("filter_compact_sharded", lens, 8);
  YATT_ALIGNED("filter_compact_sharded", new_cu, 8);
  YATT_ALIGNED("filter_compact_sharded", counts, 8);
  YATT_ALIGNED("filter_compact_sharded", ws, 8);
  YATT_ALIGNED("filter_compact_sharded", d_all_records, 8);
  return filter_compact_launch(r, lens, n, first_sample_id, G, d_all_records, world, keep, map,
                               new_cu, counts, ws, ws_bytes, as_stream(stream));
}

int yatt_gather_varlen(const void* src, const int64_t* old_cu, const int32_t* map,
                       const int64_t* new_cu, const int64_t* d_n_kept, int64_t max_kept,
                       const int64_t* d_dst_offset, int32_t elem_bytes, void* dst, void* stream) {
  YATT_ALIGNED("gather_varlen", old_cu, 8);
  YATT_ALIGNED("gather_varlen", map, 4);
  YATT_ALIGNED("gather_varlen", new_cu, 8);
  YATT_ALIGNED("gather_varlen", d_n_kept, 8);
  YATT_ALIGNED("gather_varlen", d_dst_offset, 8);
  return gather_varlen_launch(src, old_cu, map, new_cu, d_n_kept, max_kept, d_dst_offset,
                              elem_bytes, dst, as_stream(stream));
}

int yatt_gather_varlen_multi(int32_t n_arrays, const void* const* srcs, void* const* dsts,
                             const int32_t* esz, const int64_t* old_cu, const int32_t* map,
                             const int64_t* new_cu, const int64_t* d_n_kept, int64_t max_kept,
                             const int64_t* d_dst_offset, void* stream) {
  YATT_ALIGNED("gather_varlen_multi", old_cu, 8);
  YATT_ALIGNED("gather_varlen_multi", map, 4);
  YATT_ALIGNED("gather_varlen_multi", new_cu, 8);
  YATT_ALIGNED("gather_varlen_multi", d_n_kept, 8);
  YATT_ALIGNED("gather_varlen_multi", d_dst_offset, 8);
  return gather_varlen_multi_launch(n_arrays, srcs, dsts, esz, old_cu, map, new_cu, d_n_kept,
                                    max_kept, d_dst_offset, as_stream(stream));
}

int yatt_gather_rows(const void* src, const int32_t* map, const int64_t* d_n_kept,
                     int64_t max_kept, int64_t row_bytes, const int64_t* d_dst_offset, void* dst,
                     void* stream) {
  YATT_ALIGNED("gather_rows", map, 4);
  YATT_ALIGNED("gather_rows", d_n_kept, 8);
  YATT_ALIGNED("gather_rows", d_dst_offset, 8);
  return gather_rows_launch(src, map, d_n_kept, max_kept, row_bytes, d_dst_offset, dst,
                            as_stream(stream));
}

int yatt_microbatch_aggregates(const int32_t* plen, const int32_t* olen, const int64_t* d_n,
                               int64_t n, int32_t mb, int32_t rank, yatt_mb_agg* out,
                               void* stream) {
  YATT_ALIGNED4("microbatch_aggregates", plen, olen, nullptr, nullptr);
  YATT_ALIGNED("microbatch_aggregates", d_n, 8);
  YATT_ALIGNED("microbatch_aggregates", out, 8);
  return microbatch_launch(plen, olen, d_n, n, mb, rank, out, as_stream(stream));
}

int yatt_exclusive_offset(const int64_t* d_counts, int32_t nranks, int32_t rank, int32_t stride,
                          int32_t field, int64_t* d_out, void* stream) {
  YATT_ALIGNED("exclusive_offset", d_counts, 8);
  YATT_ALIGNED("exclusive_offset", d_out, 8);
  return exclusive_offset_launch(d_counts, nranks, rank, stride, field, d_out, as_stream(stream));
}

size_t yatt_sort_order_workspace_bytes(int64_t n) { return sort_workspace_bytes(n); }

int yatt_sort_order_desc(const int32_t* len, int64_t n, uint32_t* order, void* ws,
                         size_t ws_bytes, void* stream) {
  YATT_ALIGNED4("sort_order_desc", len, order, nullptr, nullptr);
  YATT_ALIGNED("sort_order_desc", ws, 8);
  return sort_order_launch(len, n, order, ws, ws_bytes, as_stream(stream));
}

int yatt_sort_and_bucket_host(const int32_t* h_len, int64_t n, int32_t B, uint64_t seed,
                              uint32_t* h_flat, int64_t* h_off) {
  YATT_REQUIRE(B > 0, YATT_ERR_CONFIG, "batch_size must be positive");
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "sort_and_bucket: n must be >= 0");
  std::vector<uint32_t> order(static_cast<size_t>(n));
  if (n > 0) {
    static thread_local DevBuf dlen, dord, dws;
    int rc = dlen.reserve(size_t(n) * 4);
    if (!rc) rc = dord.reserve(size_t(n) * 4);
    if (!rc) rc = dws.reserve(sort_workspace_bytes(n));
    if (rc) return rc;
    cudaStream_t st = nullptr;
    YATT_TRY_CUDA(cudaMemcpyAsync(dlen.p, h_len, size_t(n) * 4, cudaMemcpyHostToDevice, st));
    rc = sort_order_launch(static_cast<int32_t*>(dlen.p), n, static_cast<uint32_t*>(dord.p), dws.p,
                           dws.bytes, st);
    if (rc) return rc;
    YATT_TRY_CUDA(cudaMemcpyAsync(order.data(), dord.p, size_t(n) * 4, cudaMemcpyDeviceToHost, st));
    YATT_TRY_CUDA(cudaStreamSynchronize(st));
  }
  // Bucket cut + bucket-order shuffle on the host (balancer.cpp:30-39):
  // std::shuffle over bucket indices with the same engine and seed permutes
  // exactly like shuffling the bucket vectors themselves.
  const int64_t nb = (n + B - 1) / B;
  std::vector<int64_t> perm(static_cast<size_t>(nb));
  std::iota(perm.begin(), perm.end(), int64_t(0));
  std::mt19937_64 rng(seed);
  std::shuffle(perm.begin(), perm.end(), rng);
  int64_t pos = 0;
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t b = perm[size_t(k)] * B, e = min64(n, b + B);
    if (h_off) h_off[k] = pos;
    for (int64_t i = b; i < e; ++i) h_flat[pos++] = order[size_t(i)];
  }
  if (h_off) h_off[nb] = pos;
  return YATT_OK;
}

int yatt_synth_logits(uint64_t seed, int64_t row0, int64_t rows, int32_t vocab, uint16_t* pol,
                      uint16_t* ref, int32_t* tgt, void* stream) {
  YATT_ALIGNED("synth_logits", pol, 16);
  YATT_ALIGNED("synth_logits", ref, 16);
  YATT_ALIGNED("synth_logits", tgt, 4);
  return synth_logits_launch(seed, row0, rows, vocab, pol, ref, tgt, as_stream(stream));
}

int yatt_synth_floats(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n, int32_t kind,
                      int32_t group_size, const float* base, float* out, void* stream) {
  YATT_ALIGNED4("synth_floats", base, out, nullptr, nullptr);
  return synth_floats_launch(seed, stream_id, i0, n, kind, group_size, base, out,
                             as_stream(stream));
}

}  // extern "C"
