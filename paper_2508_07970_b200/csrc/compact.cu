// compact.cu — A5 dynamic-sampling filter + A6 survivor compaction/repack,
// and R4 microbatch aggregates.  Integer work, bit-exact.
//
// Reference semantics being kept:
//  * survivors keep their relative (sample-id) order, exactly like the
//    ordered pending compaction of shard_round_output
//    (proj/src/simcore.cpp:167-177) and the rank-order concatenation of
//    copy_back (simcore.cpp:107-119);
//  * microbatches are consecutive runs of `microbatch_size` survivors with
//    {count, max response length, sum(prompt+response)}
//    (build_microbatches, simcore.cpp:17-39);
//  * the group filter is DAPO's zero-variance rule: a group
//    whose rewards are all bitwise identical carries no advantage signal.
// Scan: reduce-then-scan over 4096-sample tiles (3 launches, deterministic).
// Gathers: one CTA per kept sample, coalesced element copies (HBM-bound).
#include <cuda_runtime.h>

#include "common.cuh"

namespace yattb {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kGatherThreads = 256;  // gather_varlen_kernel block size
constexpr int kScanPerThread = 4;
constexpr int kScanTile = kScanThreads * kScanPerThread;

__global__ void group_filter_kernel(const float* r, int64_t n, int32_t G, uint8_t* keep) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t ng = n / G;
  if (g >= ng) return;
  const uint32_t* bits = reinterpret_cast<const uint32_t*>(r) + g * G;
  const uint32_t b0 = bits[0];
  uint8_t k = 0;
  for (int i = 1; i < G; ++i) k |= (bits[i] != b0);
  keep[g] = k;
}

// Block-wide exclusive scan of int64 pairs (samples, tokens); returns totals.
struct Pair {
  int64_t a, b;
};
__device__ __forceinline__ Pair block_exclusive_scan(Pair x, Pair* total) {
  __shared__ int64_t sa[kScanThreads / 32], sb[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Pair inc = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t oa = __shfl_up_sync(0xffffffffu, inc.a, d);
    const int64_t ob = __shfl_up_sync(0xffffffffu, inc.b, d);
    if (lane >= d) {
      inc.a += oa;
      inc.b += ob;
    }
  }
  if (lane == 31) {
    sa[w] = inc.a;
    sb[w] = inc.b;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    int64_t va = lane < nw ? sa[lane] : 0, vb = lane < nw ? sb[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t oa = __shfl_up_sync(0xffffffffu, va, d);
      const int64_t ob = __shfl_up_sync(0xffffffffu, vb, d);
      if (lane >= d) {
        va += oa;
        vb += ob;
      }
    }
    if (lane < nw) {
      sa[lane] = va;
      sb[lane] = vb;
    }
  }
  __syncthreads();
  const int64_t wa = w > 0 ? sa[w - 1] : 0, wb = w > 0 ? sb[w - 1] : 0;
  total->a = sa[(blockDim.x >> 5) - 1];
  total->b = sb[(blockDim.x >> 5) - 1];
  __syncthreads();
  return Pair{wa + inc.a - x.a, wb + inc.b - x.b};
}

// Pass 1: per-tile kept (samples, tokens).
__global__ void __launch_bounds__(kScanThreads) compact_count_kernel(
    const uint8_t* keep, const int64_t* lens, int64_t n, int32_t G, int64_t* tile_tot) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanPerThread;
  Pair x{0, 0};
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const int64_t i = base + k;
    if (i < n && keep[i / G]) {
      x.a += 1;
      x.b += lens[i];
    }
  }
  Pair tot;
  block_exclusive_scan(x, &tot);
  if (threadIdx.x == 0) {
    tile_tot[2 * blockIdx.x] = tot.a;
    tile_tot[2 * blockIdx.x + 1] = tot.b;
  }
}

// Pass 2: exclusive scan of tile totals (single CTA, sequential chunks).
__global__ void __launch_bounds__(kScanThreads) compact_tiles_kernel(
    int64_t* tile_tot, int64_t ntiles, int64_t n_groups, const uint8_t* keep, int64_t* new_cu,
    int64_t* counts) {
  Pair carry{0, 0};
  for (int64_t b0 = 0; b0 < ntiles; b0 += kScanThreads) {
    const int64_t t = b0 + threadIdx.x;
    Pair x{0, 0};
    if (t < ntiles) x = Pair{tile_tot[2 * t], tile_tot[2 * t + 1]};
    Pair tot;
    const Pair ex = block_exclusive_scan(x, &tot);
    if (t < ntiles) {
      tile_tot[2 * t] = carry.a + ex.a;
      tile_tot[2 * t + 1] = carry.b + ex.b;
    }
    carry.a += tot.a;
    carry.b += tot.b;
  }
  // kept groups
  int64_t kg = 0;
  for (int64_t g = threadIdx.x; g < n_groups; g += kScanThreads) kg += keep[g];
  __shared__ int64_t red[kScanThreads / 32];
  kg = warp_sum(kg);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = kg;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int i = 0; i < kScanThreads / 32; ++i) s += red[i];
    counts[0] = carry.a;
    counts[1] = carry.b;
    counts[2] = s;
    new_cu[carry.a] = carry.b;
  }
}

// Pass 3: scatter index map and packed offsets.
__global__ void __launch_bounds__(kScanThreads) compact_scatter_kernel(
    const uint8_t* keep, const int64_t* lens, int64_t n, int32_t G, const int64_t* tile_off,
    int32_t* index_map, int64_t* new_cu) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanPerThread;
  Pair x{0, 0};
  bool kk[kScanPerThread];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const int64_t i = base + k;
    kk[k] = i < n && keep[i / G];
    if (kk[k]) {
      x.a += 1;
      x.b += lens[i];
    }
  }
  Pair tot;
  Pair ex = block_exclusive_scan(x, &tot);
  ex.a += tile_off[2 * blockIdx.x];
  ex.b += tile_off[2 * blockIdx.x + 1];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    if (!kk[k]) continue;
    const int64_t i = base + k;
    index_map[ex.a] = int32_t(i);
    new_cu[ex.a] = ex.b;
    ex.a += 1;
    ex.b += lens[i];
  }
}

template <typename T>
__global__ void gather_varlen_kernel(const T* src, const int64_t* old_cu, const int32_t* map,
                                     const int64_t* new_cu, const int64_t* n_kept,
                                     const int64_t* dst_off, T* dst) {
  const int64_t nk = *n_kept;
  const int64_t off = dst_off ? *dst_off : 0;
  for (int64_t j = blockIdx.x; j < nk; j += gridDim.x) {
    const int32_t s = map[j];
    const int64_t b = old_cu[s], len = old_cu[s + 1] - b;
    const T* sp = src + b;
    T* dp = dst + (new_cu[j] + off);
    // 8 independent coalesced loads in flight per thread before the stores
    constexpr int kU = 8, kB = kGatherThreads;
    int64_t k = threadIdx.x;
    for (; k + (kU - 1) * kB < len; k += kU * kB) {
      T v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = __ldg(sp + k + u * kB);
#pragma unroll
      for (int u = 0; u < kU; ++u) dp[k + u * kB] = v[u];
    }
    for (; k < len; k += kB) dp[k] = __ldg(sp + k);
  }
}

__global__ void gather_rows_kernel(const uint8_t* src, const int32_t* map, const int64_t* n_kept,
                                   int64_t row_bytes, const int64_t* dst_off, uint8_t* dst) {
  const int64_t nk = *n_kept;
  const int64_t off = dst_off ? *dst_off : 0;
  for (int64_t j = blockIdx.x; j < nk; j += gridDim.x) {
    const uint8_t* sp = src + int64_t(map[j]) * row_bytes;
    uint8_t* dp = dst + (j + off) * row_bytes;
    for (int64_t k = threadIdx.x; k < row_bytes; k += blockDim.x) dp[k] = sp[k];
  }
}

__global__ void microbatch_kernel(const int32_t* plen, const int32_t* olen, const int64_t* n_ptr,
                                  int64_t n_host, int32_t mb, int32_t rank, yatt_mb_agg* out) {
  const int64_t n = n_ptr ? *n_ptr : n_host;
  const int64_t nmb = (n + mb - 1) / mb;
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nmb) return;
  yatt_mb_agg a{rank, int32_t(k), 0, 0, 0};
  for (int64_t i = k * mb; i < min64(n, (k + 1) * mb); ++i) {
    a.sample_count += 1;
    a.max_out_len_tokens = max(a.max_out_len_tokens, olen[i]);
    a.score_tokens += int64_t(plen[i]) + int64_t(olen[i]);
  }
  out[k] = a;
}

__global__ void exclusive_offset_kernel(const int64_t* counts, int32_t nranks, int32_t rank,
                                        int32_t stride, int32_t field, int64_t* out) {
  if (threadIdx.x != 0) return;
  int64_t s = 0;
  for (int r = 0; r < rank && r < nranks; ++r) s += counts[int64_t(r) * stride + field];
  *out = s;
}

}  // namespace

size_t compact_workspace_bytes(int64_t n) {
  return size_t(2 * ceil_div(n > 0 ? n : 1, kScanTile)) * sizeof(int64_t);
}

int filter_compact_launch(const float* r, const int64_t* lens, int64_t n, int32_t G,
                          uint8_t* keep, int32_t* map, int64_t* new_cu, int64_t* counts, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  YATT_REQUIRE(G > 0, YATT_ERR_CONFIG, "filter_compact: group_size must be positive");
  YATT_REQUIRE(n >= 0 && n % G == 0, YATT_ERR_CONFIG,
               "filter_compact: n_samples (%lld) must be a multiple of group_size (%d)",
               (long long)n, G);
  YATT_REQUIRE(n < (int64_t(1) << 31), YATT_ERR_CONFIG, "filter_compact: too many samples");
  YATT_REQUIRE(ws != nullptr && ws_bytes >= compact_workspace_bytes(n), YATT_ERR_WORKSPACE,
               "filter_compact: workspace too small");
  const int64_t ng = n / G;
  if (ng > 0) {
    group_filter_kernel<<<unsigned(ceil_div(ng, 256)), 256, 0, st>>>(r, n, G, keep);
    int rc = check_launch("group_filter_kernel");
    if (rc) return rc;
  }
  const int64_t ntiles = ceil_div(n, kScanTile);
  int64_t* tiles = static_cast<int64_t*>(ws);
  if (ntiles > 0) {
    compact_count_kernel<<<unsigned(ntiles), kScanThreads, 0, st>>>(keep, lens, n, G, tiles);
    int rc = check_launch("compact_count_kernel");
    if (rc) return rc;
  }
  compact_tiles_kernel<<<1, kScanThreads, 0, st>>>(tiles, ntiles, ng, keep, new_cu, counts);
  int rc = check_launch("compact_tiles_kernel");
  if (rc) return rc;
  if (ntiles > 0) {
    compact_scatter_kernel<<<unsigned(ntiles), kScanThreads, 0, st>>>(keep, lens, n, G, tiles,
                                                                      map, new_cu);
    rc = check_launch("compact_scatter_kernel");
  }
  return rc;
}

int gather_varlen_launch(const void* src, const int64_t* old_cu, const int32_t* map,
                         const int64_t* new_cu, const int64_t* n_kept, int64_t max_kept,
                         const int64_t* dst_off, int32_t elem_bytes, void* dst, cudaStream_t st) {
  YATT_REQUIRE(max_kept >= 0, YATT_ERR_CONFIG, "gather_varlen: max_kept must be >= 0");
  if (max_kept == 0) return YATT_OK;
  const int grid = int(min64(max_kept, int64_t(num_sms()) * 16));
  switch (elem_bytes) {
    case 1:
      gather_varlen_kernel<uint8_t><<<grid, 256, 0, st>>>(
          static_cast<const uint8_t*>(src), old_cu, map, new_cu, n_kept, dst_off,
          static_cast<uint8_t*>(dst));
      break;
    case 2:
      gather_varlen_kernel<uint16_t><<<grid, 256, 0, st>>>(
          static_cast<const uint16_t*>(src), old_cu, map, new_cu, n_kept, dst_off,
          static_cast<uint16_t*>(dst));
      break;
    case 4:
      gather_varlen_kernel<uint32_t><<<grid, 256, 0, st>>>(
          static_cast<const uint32_t*>(src), old_cu, map, new_cu, n_kept, dst_off,
          static_cast<uint32_t*>(dst));
      break;
    case 8:
      gather_varlen_kernel<uint64_t><<<grid, 256, 0, st>>>(
          static_cast<const uint64_t*>(src), old_cu, map, new_cu, n_kept, dst_off,
          static_cast<uint64_t*>(dst));
      break;
    default:
      return set_error(YATT_ERR_CONFIG, "gather_varlen: elem_bytes must be 1, 2, 4 or 8 (got %d)",
                       elem_bytes);
  }
  return check_launch("gather_varlen_kernel");
}

int gather_rows_launch(const void* src, const int32_t* map, const int64_t* n_kept,
                       int64_t max_kept, int64_t row_bytes, const int64_t* dst_off, void* dst,
                       cudaStream_t st) {
  YATT_REQUIRE(row_bytes > 0 && max_kept >= 0, YATT_ERR_CONFIG, "gather_rows: bad sizes");
  if (max_kept == 0) return YATT_OK;
  const int grid = int(min64(max_kept, int64_t(num_sms()) * 16));
  gather_rows_kernel<<<grid, 128, 0, st>>>(static_cast<const uint8_t*>(src), map, n_kept,
                                           row_bytes, dst_off, static_cast<uint8_t*>(dst));
  return check_launch("gather_rows_kernel");
}

int microbatch_launch(const int32_t* plen, const int32_t* olen, const int64_t* d_n, int64_t n,
                      int32_t mb, int32_t rank, yatt_mb_agg* out, cudaStream_t st) {
  YATT_REQUIRE(mb > 0, YATT_ERR_CONFIG, "microbatch_size must be positive");
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "microbatch: n must be >= 0");
  const int64_t nmb = ceil_div(n, mb);
  if (nmb == 0) return YATT_OK;
  microbatch_kernel<<<unsigned(ceil_div(nmb, 128)), 128, 0, st>>>(plen, olen, d_n, n, mb, rank,
                                                                  out);
  return check_launch("microbatch_kernel");
}

int exclusive_offset_launch(const int64_t* counts, int32_t nranks, int32_t rank, int32_t stride,
                            int32_t field, int64_t* out, cudaStream_t st) {
  YATT_REQUIRE(nranks > 0 && rank >= 0 && rank < nranks, YATT_ERR_RANK,
               "exclusive_offset: rank %d out of range [0, %d)", rank, nranks);
  exclusive_offset_kernel<<<1, 32, 0, st>>>(counts, nranks, rank, stride, field, out);
  return check_launch("exclusive_offset_kernel");
}

}  // namespace yattb
