// sort_order.cu — R10: the sort half of balancer::sort_and_bucket
// (proj/src/balancer.cpp:16-36): indices ordered by length descending, ties
// broken by index ascending.  Encoded as unique 64-bit keys
//     key = (~(len ^ 0x80000000) << 32) | index
// so an ascending sort of the keys IS the reference's comparator order and
// the result is independent of sort stability.  Chunks of 4096 keys are
// bitonic-sorted in shared memory, then merged pairwise by rank (binary
// search into the partner run) until one run remains.  Bucket cutting and the
// mt19937_64 std::shuffle of bucket order stay on the host (capi.cu) so the
// permutation is bit-identical to libstdc++.
#include <cuda_runtime.h>

#include "common.cuh"

namespace yattb {
namespace {

constexpr int kChunk = 4096;
constexpr int kSortThreads = 1024;

__global__ void make_keys_kernel(const int32_t* len, int64_t n, uint64_t* keys) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t u = uint32_t(len[i]) ^ 0x80000000u;
  keys[i] = (uint64_t(~u) << 32) | uint64_t(uint32_t(i));
}

__global__ void __launch_bounds__(kSortThreads) chunk_sort_kernel(uint64_t* keys, int64_t n) {
  __shared__ uint64_t s[kChunk];
  const int64_t base = int64_t(blockIdx.x) * kChunk;
  for (int i = threadIdx.x; i < kChunk; i += kSortThreads)
    s[i] = base + i < n ? keys[base + i] : ~0ull;
  __syncthreads();
  for (int k = 2; k <= kChunk; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < kChunk; i += kSortThreads) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const uint64_t a = s[i], b = s[p];
          if ((a > b) == up) {
            s[i] = b;
            s[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < kChunk; i += kSortThreads)
    if (base + i < n) keys[base + i] = s[i];
}

__device__ __forceinline__ int64_t lower_bound(const uint64_t* a, int64_t len, uint64_t key) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void merge_pass_kernel(const uint64_t* in, uint64_t* out, int64_t n, int64_t width) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t pair = i / (2 * width);
  const int64_t a0 = pair * 2 * width;
  const int64_t b0 = min64(n, a0 + width);
  const int64_t b1 = min64(n, a0 + 2 * width);
  const uint64_t key = in[i];
  int64_t pos;
  if (i < b0) pos = a0 + (i - a0) + lower_bound(in + b0, b1 - b0, key);
  else pos = a0 + (i - b0) + lower_bound(in + a0, b0 - a0, key);
  out[pos] = key;
}

__global__ void extract_kernel(const uint64_t* keys, int64_t n, uint32_t* order) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) order[i] = uint32_t(keys[i]);
}

}  // namespace

size_t sort_workspace_bytes(int64_t n) { return size_t(2) * size_t(n > 0 ? n : 1) * 8; }

int sort_order_launch(const int32_t* len, int64_t n, uint32_t* order, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  YATT_REQUIRE(n >= 0 && n < (int64_t(1) << 32), YATT_ERR_CONFIG, "sort: n out of range");
  YATT_REQUIRE(ws != nullptr && ws_bytes >= sort_workspace_bytes(n), YATT_ERR_WORKSPACE,
               "sort: workspace too small");
  if (n == 0) return YATT_OK;
  uint64_t* a = static_cast<uint64_t*>(ws);
  uint64_t* b = a + n;
  make_keys_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(len, n, a);
  int rc = check_launch("make_keys_kernel");
  if (rc) return rc;
  chunk_sort_kernel<<<unsigned(ceil_div(n, kChunk)), kSortThreads, 0, st>>>(a, n);
  rc = check_launch("chunk_sort_kernel");
  if (rc) return rc;
  for (int64_t w = kChunk; w < n; w <<= 1) {
    merge_pass_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(a, b, n, w);
    rc = check_launch("merge_pass_kernel");
    if (rc) return rc;
    uint64_t* t = a;
    a = b;
    b = t;
  }
  extract_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(a, n, order);
  return check_launch("extract_kernel");
}

}  // namespace yattb
