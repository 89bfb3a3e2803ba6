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

// Local group k of a shard that starts at global sample first_id covers
// global group g0 + k (g0 = first_id / G), i.e. local samples
// [max(0, (g0+k)*G - first_id), min(n, (g0+k+1)*G - first_id)); the first and
// last local groups may be partial when groups straddle ranks (sample-level
// shard_dataset, workload.cpp:183-198).  keep = some reward differs bitwise
// from the group's first; for a partial group the other ranks' boundary
// records (straddle.cu: {group, first reward bits, any-differs} for their
// first and last local groups) are folded in, so every rank holding a piece
// of the group takes the same exact decision.
struct FilterRecord {
  int64_t g, bits, anydiff;
};

__global__ void group_filter_kernel(const float* r, int64_t n, uint64_t first_id, int32_t G,
                                    int64_t ng, const int64_t* recs, int32_t world,
                                    uint8_t* keep) {
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= ng) return;
  const uint64_t g = first_id / uint64_t(G) + uint64_t(k);
  const int64_t lo = max64(0, int64_t(g * uint64_t(G)) - int64_t(first_id));
  const int64_t hi = min64(n, int64_t((g + 1) * uint64_t(G)) - int64_t(first_id));
  const uint32_t* bits = reinterpret_cast<const uint32_t*>(r);
  const uint32_t b0 = bits[lo];
  uint8_t any = 0;
  for (int64_t i = lo + 1; i < hi; ++i) any |= (bits[i] != b0);
  if (recs != nullptr && (k == 0 || k == ng - 1)) {
    for (int32_t q = 0; q < world; ++q)
      for (int side = 0; side < 2; ++side) {
        const int64_t* rec = recs + 6 * q + 3 * side;
        if (rec[0] == int64_t(g)) any |= uint8_t(rec[2] != 0 || uint32_t(rec[1]) != b0);
      }
  }
  keep[k] = any;
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
    const uint8_t* keep, const int64_t* lens, int64_t n, int32_t G, int32_t first_mod,
    int64_t* tile_tot) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanPerThread;
  Pair x{0, 0};
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const int64_t i = base + k;
    if (i < n && keep[(first_mod + i) / G]) {
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
// kept_groups counts the groups whose FIRST sample is local (a straddling
// group is counted once, by the rank holding its start).
__global__ void __launch_bounds__(kScanThreads) compact_tiles_kernel(
    int64_t* tile_tot, int64_t ntiles, int64_t n_groups, int32_t first_mod, const uint8_t* keep,
    int64_t* new_cu, int64_t* counts) {
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
  for (int64_t g = (first_mod != 0 ? 1 : 0) + threadIdx.x; g < n_groups; g += kScanThreads)
    kg += keep[g];
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
    const uint8_t* keep, const int64_t* lens, int64_t n, int32_t G, int32_t first_mod,
    const int64_t* tile_off, int32_t* index_map, int64_t* new_cu) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanPerThread;
  Pair x{0, 0};
  bool kk[kScanPerThread];
#pragma unroll
  for (int k = 0; k < kScanPerThread; ++k) {
    const int64_t i = base + k;
    kk[k] = i < n && keep[(first_mod + i) / G];
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

// ---- byte-exact gathers ---------------------------------------------------
__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
// bytes [s, s+16) of the 32-byte window (a ++ b), s in [0, 16)
__device__ __forceinline__ uint4 window16(const uint4& a, const uint4& b, int s) {
  const uint32_t r = uint32_t(s & 3) * 8u;
  switch (s >> 2) {
    case 0:
      return make_uint4(__funnelshift_r(a.x, a.y, r), __funnelshift_r(a.y, a.z, r),
                        __funnelshift_r(a.z, a.w, r), __funnelshift_r(a.w, b.x, r));
    case 1:
      return make_uint4(__funnelshift_r(a.y, a.z, r), __funnelshift_r(a.z, a.w, r),
                        __funnelshift_r(a.w, b.x, r), __funnelshift_r(b.x, b.y, r));
    case 2:
      return make_uint4(__funnelshift_r(a.z, a.w, r), __funnelshift_r(a.w, b.x, r),
                        __funnelshift_r(b.x, b.y, r), __funnelshift_r(b.y, b.z, r));
    default:
      return make_uint4(__funnelshift_r(a.w, b.x, r), __funnelshift_r(b.x, b.y, r),
                        __funnelshift_r(b.y, b.z, r), __funnelshift_r(b.z, b.w, r));
  }
}
__device__ __forceinline__ uint4 shfl_down16(const uint4& v) {
  return make_uint4(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1),
                    __shfl_down_sync(0xffffffffu, v.z, 1), __shfl_down_sync(0xffffffffu, v.w, 1));
}

// One CTA copies L bytes src -> dst for any relative alignment: bytewise
// head up to dst's first 16-B boundary, then aligned 16-B stores; each lane
// loads one ALIGNED 16-B source chunk, takes its right neighbour's chunk by
// shuffle (the last lane loads it) and funnel-shifts the 16 bytes it needs
// out of the 32-byte window.  Loads touch only aligned chunks holding needed
// bytes; four 512-B groups per warp are in flight per iteration.
__device__ __forceinline__ void cta_copy_bytes(const uint8_t* src, uint8_t* dst, int64_t L) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t head = min64(L, int64_t((16u - (reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u));
  const int64_t nch = (L - head) >> 4;
  const int64_t tail0 = head + nch * 16;
  if (tid < head) dst[tid] = src[tid];
  if (tid < L - tail0) dst[tail0 + tid] = src[tail0 + tid];
  const uint8_t* s0 = src + head;
  uint8_t* d0 = dst + head;
  const int sh = int(reinterpret_cast<uintptr_t>(s0) & 15u);
  const uint8_t* sb = s0 - sh;  // aligned
  // chunk nch (when sh != 0) holds the last body chunk's final sh bytes
  const int64_t nload = nch + (sh != 0 ? 1 : 0);
  constexpr int kU = 4;
  for (int64_t g0 = int64_t(warp) * 32 * kU; g0 < nch; g0 += int64_t(nwarps) * 32 * kU) {
    uint4 a[kU], b[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t c = g0 + u * 32 + lane;
      a[u] = c < nload ? ldg16(sb + 16 * c) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      b[u] = shfl_down16(a[u]);
      const int64_t c = g0 + u * 32 + lane;
      if (lane == 31 && sh != 0 && c < nch) b[u] = ldg16(sb + 16 * (c + 1));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t c = g0 + u * 32 + lane;
      if (c < nch) *reinterpret_cast<uint4*>(d0 + 16 * c) = sh ? window16(a[u], b[u], sh) : a[u];
    }
  }
}

struct GatherArrays {
  const uint8_t* src[YATT_GATHER_MAX_ARRAYS];
  uint8_t* dst[YATT_GATHER_MAX_ARRAYS];
  int32_t esz[YATT_GATHER_MAX_ARRAYS];
  int32_t n;
};

// One CTA per kept sample (grid-stride), all arrays of the sample in turn;
// thread 0 fetches the NEXT sample's (map -> old_cu, new_cu) chain while the
// current one is copied.
__global__ void __launch_bounds__(kGatherThreads) gather_varlen_kernel(
    const GatherArrays arr, const int64_t* old_cu, const int32_t* map, const int64_t* new_cu,
    const int64_t* n_kept, const int64_t* dst_off) {
  __shared__ int64_t meta[2][3];  // src element offset, length, dst element offset
  const int64_t nk = *n_kept;
  const int64_t off = dst_off ? *dst_off : 0;
  auto fetch = [&](int64_t j, int64_t* m) {
    const int32_t s = __ldg(map + j);
    const int64_t b = __ldg(old_cu + s);
    m[0] = b;
    m[1] = __ldg(old_cu + s + 1) - b;
    m[2] = __ldg(new_cu + j) + off;
  };
  int64_t j = blockIdx.x;
  if (threadIdx.x == 0 && j < nk) fetch(j, meta[0]);
  __syncthreads();
  for (int buf = 0; j < nk; j += gridDim.x, buf ^= 1) {
    int64_t nxt[3];
    const bool more = j + gridDim.x < nk;
    if (threadIdx.x == 0 && more) fetch(j + gridDim.x, nxt);  // in flight during the copy
    for (int a = 0; a < arr.n; ++a) {
      const int64_t e = arr.esz[a];
      cta_copy_bytes(arr.src[a] + meta[buf][0] * e, arr.dst[a] + meta[buf][2] * e, meta[buf][1] * e);
    }
    if (threadIdx.x == 0 && more) {
      meta[buf ^ 1][0] = nxt[0];
      meta[buf ^ 1][1] = nxt[1];
      meta[buf ^ 1][2] = nxt[2];
    }
    __syncthreads();
  }
}

// Rows: flattened over (kept row, w-byte word), w = widest of 16/8/4/1 that
// divides row_bytes and both base alignments.
template <typename W>
__global__ void gather_rows_kernel(const uint8_t* src, const int32_t* map, const int64_t* n_kept,
                                   int64_t words_per_row, const int64_t* dst_off, uint8_t* dst) {
  const int64_t nk = *n_kept;
  const int64_t off = dst_off ? *dst_off : 0;
  const W* s = reinterpret_cast<const W*>(src);
  W* d = reinterpret_cast<W*>(dst);
  const int64_t total = nk * words_per_row;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = i / words_per_row, w = i - j * words_per_row;
    d[(j + off) * words_per_row + w] = s[int64_t(map[j]) * words_per_row + w];
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

int filter_compact_launch(const float* r, const int64_t* lens, int64_t n, uint64_t first_id,
                          int32_t G, const int64_t* recs, int32_t world, uint8_t* keep,
                          int32_t* map, int64_t* new_cu, int64_t* counts, void* ws,
                          size_t ws_bytes, cudaStream_t st) {
  YATT_REQUIRE(G > 0, YATT_ERR_CONFIG, "filter_compact: group_size must be positive");
  YATT_REQUIRE(n >= 0, YATT_ERR_CONFIG, "filter_compact: n_samples must be >= 0");
  YATT_REQUIRE(n < (int64_t(1) << 31), YATT_ERR_CONFIG, "filter_compact: too many samples");
  YATT_REQUIRE(recs == nullptr || (world >= 1 && world <= 4096), YATT_ERR_CONFIG,
               "filter_compact: world must be in [1, 4096] with boundary records");
  YATT_REQUIRE(ws != nullptr && ws_bytes >= compact_workspace_bytes(n), YATT_ERR_WORKSPACE,
               "filter_compact: workspace too small");
  const int64_t ng = n > 0 ? int64_t((first_id + uint64_t(n) - 1) / uint64_t(G) -
                                     first_id / uint64_t(G) + 1) : 0;
  const int32_t first_mod = int32_t(first_id % uint64_t(G));
  if (ng > 0) {
    group_filter_kernel<<<unsigned(ceil_div(ng, 256)), 256, 0, st>>>(r, n, first_id, G, ng, recs,
                                                                     world, keep);
    int rc = check_launch("group_filter_kernel");
    if (rc) return rc;
  }
  const int64_t ntiles = ceil_div(n, kScanTile);
  int64_t* tiles = static_cast<int64_t*>(ws);
  if (ntiles > 0) {
    compact_count_kernel<<<unsigned(ntiles), kScanThreads, 0, st>>>(keep, lens, n, G, first_mod,
                                                                    tiles);
    int rc = check_launch("compact_count_kernel");
    if (rc) return rc;
  }
  compact_tiles_kernel<<<1, kScanThreads, 0, st>>>(tiles, ntiles, ng, first_mod, keep, new_cu,
                                                   counts);
  int rc = check_launch("compact_tiles_kernel");
  if (rc) return rc;
  if (ntiles > 0) {
    compact_scatter_kernel<<<unsigned(ntiles), kScanThreads, 0, st>>>(keep, lens, n, G, first_mod,
                                                                      tiles, map, new_cu);
    rc = check_launch("compact_scatter_kernel");
  }
  return rc;
}

// One boundary record {g, first reward bits, any-differs} x {first, last
// local group}: what the other ranks need to decide a straddling group.
__global__ void filter_record_kernel(const float* r, int64_t n, uint64_t first_id, int32_t G,
                                     int64_t* rec) {
  const uint32_t* bits = reinterpret_cast<const uint32_t*>(r);
  const uint64_t g0 = first_id / uint64_t(G);
  const uint64_t g1 = (first_id + uint64_t(n) - 1) / uint64_t(G);
  for (int side = 0; side < 2; ++side) {
    const uint64_t g = side == 0 ? g0 : g1;
    const int64_t lo = max64(0, int64_t(g * uint64_t(G)) - int64_t(first_id));
    const int64_t hi = min64(n, int64_t((g + 1) * uint64_t(G)) - int64_t(first_id));
    const uint32_t b0 = bits[lo];
    int any = 0;
    for (int64_t i = lo + 1 + threadIdx.x; i < hi; i += blockDim.x) any |= (bits[i] != b0);
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) {
      rec[3 * side + 0] = int64_t(g);
      rec[3 * side + 1] = int64_t(b0);
      rec[3 * side + 2] = any;
    }
  }
}

int filter_record_launch(const float* r, int64_t n, uint64_t first_id, int32_t G, int64_t* rec,
                         cudaStream_t st) {
  YATT_REQUIRE(G > 0, YATT_ERR_CONFIG, "filter_boundary_record: group_size must be positive");
  YATT_REQUIRE(rec != nullptr, YATT_ERR_CONFIG, "filter_boundary_record: null record");
  if (n <= 0) {  // an empty shard holds no group: a record matching nothing
    const int64_t none[6] = {-1, 0, 0, -1, 0, 0};
    YATT_TRY_CUDA(cudaMemcpyAsync(rec, none, sizeof(none), cudaMemcpyHostToDevice, st));
    return YATT_OK;
  }
  filter_record_kernel<<<1, 256, 0, st>>>(r, n, first_id, G, rec);
  return check_launch("filter_record_kernel");
}

int gather_varlen_multi_launch(int32_t n_arrays, const void* const* srcs, void* const* dsts,
                               const int32_t* esz, const int64_t* old_cu, const int32_t* map,
                               const int64_t* new_cu, const int64_t* n_kept, int64_t max_kept,
                               const int64_t* dst_off, cudaStream_t st) {
  YATT_REQUIRE(max_kept >= 0, YATT_ERR_CONFIG, "gather_varlen: max_kept must be >= 0");
  YATT_REQUIRE(n_arrays >= 1 && n_arrays <= YATT_GATHER_MAX_ARRAYS, YATT_ERR_CONFIG,
               "gather_varlen: n_arrays must be in [1, %d] (got %d)", YATT_GATHER_MAX_ARRAYS,
               n_arrays);
  YATT_REQUIRE(srcs && dsts && esz, YATT_ERR_CONFIG, "gather_varlen: null array list");
  GatherArrays arr{};
  arr.n = n_arrays;
  for (int a = 0; a < n_arrays; ++a) {
    YATT_REQUIRE(esz[a] == 1 || esz[a] == 2 || esz[a] == 4 || esz[a] == 8, YATT_ERR_CONFIG,
                 "gather_varlen: elem_bytes must be 1, 2, 4 or 8 (got %d)", esz[a]);
    YATT_REQUIRE((reinterpret_cast<uintptr_t>(srcs[a]) % uintptr_t(esz[a])) == 0 &&
                     (reinterpret_cast<uintptr_t>(dsts[a]) % uintptr_t(esz[a])) == 0,
                 YATT_ERR_CONFIG, "gather_varlen: array %d not aligned to its element size", a);
    arr.src[a] = static_cast<const uint8_t*>(srcs[a]);
    arr.dst[a] = static_cast<uint8_t*>(dsts[a]);
    arr.esz[a] = esz[a];
  }
  if (max_kept == 0) return YATT_OK;
  // ~one CTA per sample: the block scheduler balances the ragged lengths
  const int grid = int(min64(max_kept, int64_t(num_sms()) * 64));
  gather_varlen_kernel<<<grid, kGatherThreads, 0, st>>>(arr, old_cu, map, new_cu, n_kept, dst_off);
  return check_launch("gather_varlen_kernel");
}

int gather_varlen_launch(const void* src, const int64_t* old_cu, const int32_t* map,
                         const int64_t* new_cu, const int64_t* n_kept, int64_t max_kept,
                         const int64_t* dst_off, int32_t elem_bytes, void* dst, cudaStream_t st) {
  void* d = dst;
  return gather_varlen_multi_launch(1, &src, &d, &elem_bytes, old_cu, map, new_cu, n_kept,
                                    max_kept, dst_off, st);
}

int gather_rows_launch(const void* src, const int32_t* map, const int64_t* n_kept,
                       int64_t max_kept, int64_t row_bytes, const int64_t* dst_off, void* dst,
                       cudaStream_t st) {
  YATT_REQUIRE(row_bytes > 0 && max_kept >= 0, YATT_ERR_CONFIG, "gather_rows: bad sizes");
  if (max_kept == 0) return YATT_OK;
  const uintptr_t al = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                       uintptr_t(row_bytes);
  const int w = (al & 15) == 0 ? 16 : (al & 7) == 0 ? 8 : (al & 3) == 0 ? 4 : 1;
  const int64_t wpr = row_bytes / w;
  const int grid = int(max64(1, min64(ceil_div(max_kept * wpr, 256), int64_t(num_sms()) * 8)));
  const uint8_t* s8 = static_cast<const uint8_t*>(src);
  uint8_t* d8 = static_cast<uint8_t*>(dst);
  switch (w) {
    case 16: gather_rows_kernel<uint4><<<grid, 256, 0, st>>>(s8, map, n_kept, wpr, dst_off, d8); break;
    case 8: gather_rows_kernel<uint2><<<grid, 256, 0, st>>>(s8, map, n_kept, wpr, dst_off, d8); break;
    case 4: gather_rows_kernel<uint32_t><<<grid, 256, 0, st>>>(s8, map, n_kept, wpr, dst_off, d8); break;
    default: gather_rows_kernel<uint8_t><<<grid, 256, 0, st>>>(s8, map, n_kept, wpr, dst_off, d8);
  }
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
