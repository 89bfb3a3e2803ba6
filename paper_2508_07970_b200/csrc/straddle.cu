// straddle.cu — prompt groups split across controller ranks.
//
// The reference shards at SAMPLE level (workload::shard_dataset,
// proj/src/workload.cpp:183-198) while the per-group unit is
// sample_id / group_size on global ids (workload.cpp:158-160).  Whenever the
// shard size is not a multiple of the group size (P = 3 or 7 at the BASELINE
// shapes, SURVEY.md §7 hard part 5) a group straddles two (or more) ranks,
// and the two group-level ops of the experience step need the other ranks'
// pieces of it:
//   * GRPO advantages: the group's (n, mean, M2) moments.  Each rank sends
//     the fp64 moments of its first and last local group (one 8-double
//     record), every rank merges all pieces of its boundary groups in rank
//     order (Chan et al.), so all ranks hold the identical table.
//   * the zero-variance filter: exact, {first reward bits, any-differs} per
//     boundary piece (compact.cu group_filter_kernel folds them in).
// Records travel through the NVLink peer all-gather kernel
// (yatt_peer_allgather_i64, one launch) or any all-gather the caller has
// (NCCL: yatt_comm_allgather_i64); the one-call yatt_peer_* entry points do
// record -> all-gather -> merge -> op on the device, stream-ordered.
#include <cuda_runtime.h>

#include "common.cuh"

namespace yattb {

int64_t grpo_num_local_groups(int64_t, uint64_t, int32_t);
int grpo_moments_launch(const float*, int64_t, uint64_t, int32_t, double*, cudaStream_t);
int grpo_adv_launch(const float*, int64_t, uint64_t, int32_t, float, int32_t, const double*,
                    float*, cudaStream_t);
size_t compact_workspace_bytes(int64_t);
int filter_compact_launch(const float*, const int64_t*, int64_t, uint64_t, int32_t,
                          const int64_t*, int32_t, uint8_t*, int32_t*, int64_t*, int64_t*, void*,
                          size_t, cudaStream_t);
int filter_record_launch(const float*, int64_t, uint64_t, int32_t, int64_t*, cudaStream_t);

namespace {

// rec = {g_first, n, mean, M2, g_last, n, mean, M2}; group ids as doubles
// (exact below 2^53); an empty shard sends g = -1.
__global__ void grpo_record_kernel(const double* mom, int64_t ng, uint64_t first_id, int32_t G,
                                   double* rec) {
  if (threadIdx.x != 0) return;
  if (ng == 0) {
    for (int q = 0; q < 8; ++q) rec[q] = q % 4 == 0 ? -1.0 : 0.0;
    return;
  }
  const uint64_t g0 = first_id / uint64_t(G);
  rec[0] = double(g0);
  rec[1] = mom[0];
  rec[2] = mom[1];
  rec[3] = mom[2];
  rec[4] = double(g0 + uint64_t(ng - 1));
  rec[5] = mom[3 * (ng - 1)];
  rec[6] = mom[3 * (ng - 1) + 1];
  rec[7] = mom[3 * (ng - 1) + 2];
}

__device__ __forceinline__ void chan_merge(double& n, double& mean, double& m2, double nb,
                                           double mb, double qb) {
  if (nb == 0.0) return;
  if (n == 0.0) {
    n = nb;
    mean = mb;
    m2 = qb;
    return;
  }
  const double nn = n + nb, d = mb - mean;
  mean = mean + d * nb / nn;
  m2 = m2 + qb + d * d * n * nb / nn;
  n = nn;
}

// Rows 0 and ng-1 of this rank's table <- the merge of every rank's piece of
// those groups, in rank order (the same order on every rank: identical bits).
__global__ void grpo_merge_kernel(double* mom, int64_t ng, uint64_t first_id, int32_t G,
                                  const double* all, int32_t world) {
  const int side = threadIdx.x;
  if (side > 1 || ng == 0 || (side == 1 && ng == 1)) return;
  const int64_t k = side == 0 ? 0 : ng - 1;
  const double g = double(first_id / uint64_t(G) + uint64_t(k));
  double n = 0, mean = 0, m2 = 0;
  for (int32_t q = 0; q < world; ++q) {
    const double* r = all + 8 * q;
    if (r[0] == g) chan_merge(n, mean, m2, r[1], r[2], r[3]);
    if (r[4] == g && r[4] != r[0]) chan_merge(n, mean, m2, r[5], r[6], r[7]);
  }
  mom[3 * k] = n;
  mom[3 * k + 1] = mean;
  mom[3 * k + 2] = m2;
}

}  // namespace

int grpo_record_launch(const double* mom, int64_t n, uint64_t first_id, int32_t G, double* rec,
                       cudaStream_t st) {
  YATT_REQUIRE(G > 0 && n >= 0 && rec != nullptr, YATT_ERR_CONFIG,
               "grpo_boundary_record: bad arguments");
  const int64_t ng = grpo_num_local_groups(n, first_id, G);
  YATT_REQUIRE(ng == 0 || mom != nullptr, YATT_ERR_CONFIG, "grpo_boundary_record: null moments");
  grpo_record_kernel<<<1, 32, 0, st>>>(mom, ng, first_id, G, rec);
  return check_launch("grpo_record_kernel");
}

int grpo_merge_launch(double* mom, int64_t n, uint64_t first_id, int32_t G, const double* all,
                      int32_t world, cudaStream_t st) {
  YATT_REQUIRE(G > 0 && n >= 0 && all != nullptr && world >= 1, YATT_ERR_CONFIG,
               "grpo_merge_boundaries: bad arguments");
  const int64_t ng = grpo_num_local_groups(n, first_id, G);
  if (ng == 0) return YATT_OK;
  YATT_REQUIRE(mom != nullptr, YATT_ERR_CONFIG, "grpo_merge_boundaries: null moments");
  grpo_merge_kernel<<<1, 32, 0, st>>>(mom, ng, first_id, G, all, world);
  return check_launch("grpo_merge_kernel");
}

}  // namespace yattb

using namespace yattb;

#define STRADDLE_ALIGNED(fn, ptr, a)                                                      \
  YATT_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & uintptr_t((a) - 1)) == 0, YATT_ERR_CONFIG, \
               "%s: %s must be %d-byte aligned", fn, #ptr, int(a))

extern "C" {

int yatt_grpo_boundary_record(const double* d_moments, int64_t n, uint64_t first_id, int32_t G,
                              double* d_record, void* stream) {
  STRADDLE_ALIGNED("grpo_boundary_record", d_moments, 8);
  STRADDLE_ALIGNED("grpo_boundary_record", d_record, 8);
  return grpo_record_launch(d_moments, n, first_id, G, d_record, as_stream(stream));
}

int yatt_grpo_merge_boundaries(double* d_moments, int64_t n, uint64_t first_id, int32_t G,
                               const double* d_all_records, int32_t world, void* stream) {
  STRADDLE_ALIGNED("grpo_merge_boundaries", d_moments, 8);
  STRADDLE_ALIGNED("grpo_merge_boundaries", d_all_records, 8);
  return grpo_merge_launch(d_moments, n, first_id, G, d_all_records, world, as_stream(stream));
}

int yatt_filter_boundary_record(const float* d_rewards, int64_t n, uint64_t first_id, int32_t G,
                                int64_t* d_record, void* stream) {
  STRADDLE_ALIGNED("filter_boundary_record", d_rewards, 4);
  STRADDLE_ALIGNED("filter_boundary_record", d_record, 8);
  return filter_record_launch(d_rewards, n, first_id, G, d_record, as_stream(stream));
}

size_t yatt_straddle_workspace_bytes(int64_t n, uint64_t first_id, int32_t G, int32_t world) {
  const int64_t ng = G > 0 ? grpo_num_local_groups(n, first_id, G) : 0;
  const size_t moments = size_t(3 * (ng > 0 ? ng : 1)) * 8;
  return ((moments + 255) & ~size_t(255)) + 256 + size_t(world > 0 ? world : 1) * 8 * 8 +
         compact_workspace_bytes(n);
}

int yatt_peer_allgather_i64(yatt_peer_t p, const int64_t* d_in, int32_t n, int64_t* d_out,
                            void* stream);
int yatt_peer_world(yatt_peer_t p, int32_t* world, int32_t* rank);

int yatt_peer_grpo_advantages(yatt_peer_t p, const float* d_rewards, int64_t n,
                              uint64_t first_id, int32_t G, float eps, int32_t norm_by_std,
                              float* d_adv, void* d_ws, size_t ws_bytes, void* stream) {
  STRADDLE_ALIGNED("peer_grpo_advantages", d_rewards, 4);
  STRADDLE_ALIGNED("peer_grpo_advantages", d_adv, 4);
  STRADDLE_ALIGNED("peer_grpo_advantages", d_ws, 8);
  int32_t world = 0, rank = 0;
  int rc = yatt_peer_world(p, &world, &rank);
  if (rc) return rc;
  YATT_REQUIRE(d_ws != nullptr && ws_bytes >= yatt_straddle_workspace_bytes(n, first_id, G, world),
               YATT_ERR_WORKSPACE, "peer_grpo_advantages: workspace too small");
  const cudaStream_t st = as_stream(stream);
  const int64_t ng = grpo_num_local_groups(n, first_id, G);
  char* ws = static_cast<char*>(d_ws);
  double* mom = reinterpret_cast<double*>(ws);
  double* rec = reinterpret_cast<double*>(ws + ((size_t(3 * (ng > 0 ? ng : 1)) * 8 + 255) & ~size_t(255)));
  double* all = rec + 32;
  rc = grpo_moments_launch(d_rewards, n, first_id, G, mom, st);
  if (!rc) rc = grpo_record_launch(mom, n, first_id, G, rec, st);
  if (!rc) rc = yatt_peer_allgather_i64(p, reinterpret_cast<const int64_t*>(rec), 8,
                                        reinterpret_cast<int64_t*>(all), stream);
  if (!rc) rc = grpo_merge_launch(mom, n, first_id, G, all, world, st);
  if (!rc) rc = grpo_adv_launch(d_rewards, n, first_id, G, eps, norm_by_std, mom, d_adv, st);
  return rc;
}

int yatt_peer_filter_compact(yatt_peer_t p, const float* d_rewards, const int64_t* d_lens,
                             int64_t n, uint64_t first_id, int32_t G, uint8_t* d_keep,
                             int32_t* d_map, int64_t* d_new_cu, int64_t* d_counts, void* d_ws,
                             size_t ws_bytes, void* stream) {
  STRADDLE_ALIGNED("peer_filter_compact", d_rewards, 4);
  STRADDLE_ALIGNED("peer_filter_compact", d_lens, 8);
  STRADDLE_ALIGNED("peer_filter_compact", d_map, 4);
  STRADDLE_ALIGNED("peer_filter_compact", d_new_cu, 8);
  STRADDLE_ALIGNED("peer_filter_compact", d_counts, 8);
  STRADDLE_ALIGNED("peer_filter_compact", d_ws, 8);
  int32_t world = 0, rank = 0;
  int rc = yatt_peer_world(p, &world, &rank);
  if (rc) return rc;
  YATT_REQUIRE(d_ws != nullptr && ws_bytes >= yatt_straddle_workspace_bytes(n, first_id, G, world),
               YATT_ERR_WORKSPACE, "peer_filter_compact: workspace too small");
  const cudaStream_t st = as_stream(stream);
  const int64_t ng = G > 0 ? grpo_num_local_groups(n, first_id, G) : 0;
  char* ws = static_cast<char*>(d_ws);
  int64_t* rec = reinterpret_cast<int64_t*>(ws + ((size_t(3 * (ng > 0 ? ng : 1)) * 8 + 255) & ~size_t(255)));
  int64_t* all = rec + 32;
  void* scan_ws = all + 8 * world;
  rc = filter_record_launch(d_rewards, n, first_id, G, rec, st);
  if (!rc) rc = yatt_peer_allgather_i64(p, rec, 6, all, stream);
  if (!rc) rc = filter_compact_launch(d_rewards, d_lens, n, first_id, G, all, world, d_keep, d_map,
                                      d_new_cu, d_counts, scan_ws, compact_workspace_bytes(n), st);
  return rc;
}

}  // extern "C"
