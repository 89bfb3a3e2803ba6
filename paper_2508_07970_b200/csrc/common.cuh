// common.cuh — shared device/host helpers for the sm_100a experience path.
//
// Keyed RNG: bit-exact restatement of the reference's L0 primitives
// (proj/include/yatt/common.hpp:17-37) usable on host and device.
// PTX wrappers: mbarrier + cp.async.bulk (TMA bulk copy engine) used by the
// streaming kernels to stage HBM tiles into shared memory.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/yatt_cuda.h"

namespace yattb {

// ---------------------------------------------------------------------------
// Error plumbing (definitions in capi.cu)
// ---------------------------------------------------------------------------
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);

#define YATT_TRY_CUDA(expr)                                              \
  do {                                                                   \
    cudaError_t _e = (expr);                                             \
    if (_e != cudaSuccess)                                               \
      return ::yattb::set_error(YATT_ERR_CUDA, "%s: %s", #expr,          \
                                cudaGetErrorString(_e));                 \
  } while (0)

#define YATT_REQUIRE(cond, code, ...)                                    \
  do {                                                                   \
    if (!(cond)) return ::yattb::set_error((code), __VA_ARGS__);         \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Number of SMs of the current device (cached per device).
int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// function attributes live in each device's context.
int ensure_dynamic_smem(const void* kernel, int bytes);

// ---------------------------------------------------------------------------
// Keyed RNG — common.hpp:17-37 (splitmix64, hash_key, uniform_from_key)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

constexpr uint64_t kHashSeed = 0x243f6a8885a308d3ULL;

__host__ __device__ __forceinline__ uint64_t hash_mix(uint64_t h, uint64_t part) {
  return splitmix64(h ^ splitmix64(part));
}
__host__ __device__ __forceinline__ uint64_t hash3(uint64_t a, uint64_t b, uint64_t c) {
  return hash_mix(hash_mix(hash_mix(kHashSeed, a), b), c);
}
__host__ __device__ __forceinline__ uint64_t hash5(uint64_t a, uint64_t b, uint64_t c,
                                                   uint64_t d, uint64_t e) {
  return hash_mix(hash_mix(hash_mix(hash_mix(hash_mix(kHashSeed, a), b), c), d), e);
}
__host__ __device__ __forceinline__ double uniform_from_key(uint64_t key) {
  return static_cast<double>(splitmix64(key) >> 11) * 0x1.0p-53;
}

// Stream ids (workload.hpp:57-58).
constexpr uint64_t kPromptLenStream = 1;
constexpr uint64_t kOutputLenStream = 2;
constexpr uint64_t kRejectionStream = 3;

// ---------------------------------------------------------------------------
// Warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exact float -> double on the integer pipes.  F2F.F64.F32 issues to the XU
// pipe; measured per kernel (tools/bench_kernels.py, both builds): the plain
// conversion wins where XU has headroom (loss, moments, GAE), this one where
// the kernel does little else per element (whiten).  Normals and +-0 by
// rebiasing the exponent; denormals, inf and NaN take the instruction.
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t u = __float_as_uint(f), a = u & 0x7fffffffu;
  if (__builtin_expect(a - 0x00800000u >= 0x7f000000u, 0) && a != 0u) return double(f);
  const uint32_t hi = (u & 0x80000000u) | (a != 0u ? (a >> 3) + 0x38000000u : 0u);
  return __hiloint2double(int(hi), int(u << 29));
}

// Deterministic reduction of nparts partial records of kF doubles
// (part[kF*i + f]) into out[f], one 256-thread block: thread t sums parts
// t, t+256, ... in order, then a fixed-shape warp/block tree.  Same order on
// every run for a given nparts.
template <int kF>
__global__ void __launch_bounds__(256) reduce_parts_kernel(const double* part, int nparts,
                                                           double* out) {
  __shared__ double red[kF][8];
  double v[kF];
#pragma unroll
  for (int f = 0; f < kF; ++f) v[f] = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) {
#pragma unroll
    for (int f = 0; f < kF; ++f) v[f] += part[kF * i + f];
  }
  const int w = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    v[f] = warp_sum(v[f]);
    if ((threadIdx.x & 31) == 0) red[f][w] = v[f];
  }
  __syncthreads();
  if (threadIdx.x < kF) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[threadIdx.x][k];
    out[threadIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA) PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// try_wait with a suspend-time hint: the warp sleeps until the phase
// completes (or the hint expires) instead of spinning on issue slots (used
// where the kernel is issue-bound: the fused loss + gradient kernel).
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}

// L2 policy: streamed-once inputs should not displace reused lines.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk copy global -> shared through the TMA engine; completes `bytes`
// transactions on `bar`.  bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Exact 2^d for integer d (0 for d < -126): scales the online accumulators
// without rounding error.
__device__ __forceinline__ float exp2_int(int d) {
  return d < -126 ? 0.0f : __int_as_float((127 + d) << 23);
}

// bf16 pair in a 32-bit word -> two fp32 (exact).
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Round-to-nearest-even fp32 -> bf16 bits (host and device identical).
__host__ __device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  __builtin_memcpy(&u, &f, 4);
#endif
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

}  // namespace yattb
