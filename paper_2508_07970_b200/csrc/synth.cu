// synth.cu — deterministic synthetic inputs (bench + parity support).
//
// Integer-derived values, exactly reproducible by the CPU oracle
// (oracle/yatt_oracle.c, same recipe): every value comes from the reference's
// keyed RNG (proj/include/yatt/common.hpp:17-37) so host and device agree bit
// for bit.  Recipe:
//   row key   rk = hash_key({seed, 101, row});  h_v = splitmix64(rk + v)
//   policy    x_v = ((h_v >> 56) - 128) / 16                 in [-8, 7.9375]
//   ref       z_v = bf16_rne(x_v + (((h_v >> 48) & 31) - 16) / 32)
//   target    y   = splitmix64(hash_key({seed, 103, row})) % V
//   at v = y  z_y = bf16_rne(x_y +/- (8 + ((h_y >> 48) & 7)) / 32)
//             (|ref - policy| >= 1/4 at the target keeps the k3 KL
//              well-conditioned for the 1e-5 relative parity bar)
#include <cuda_runtime.h>

#include "common.cuh"

namespace yattb {
namespace {

__host__ __device__ __forceinline__ uint16_t synth_policy_bits(uint64_t h) {
  const int k = int(h >> 56) - 128;
  return f32_to_bf16_rne(float(k) * (1.0f / 16.0f));
}
__host__ __device__ __forceinline__ uint16_t synth_ref_bits(uint64_t h, bool is_target) {
  const int k = int(h >> 56) - 128;
  const float x = float(k) * (1.0f / 16.0f);
  float d;
  if (is_target) {
    const int mag = 8 + int((h >> 48) & 7);
    d = float(((h >> 47) & 1) ? mag : -mag) * (1.0f / 32.0f);
  } else {
    d = float(int((h >> 48) & 31) - 16) * (1.0f / 32.0f);
  }
  return f32_to_bf16_rne(x + d);  // x + d is exact in fp32
}

__global__ void synth_targets_kernel(uint64_t seed, int64_t row0, int64_t rows, int32_t V,
                                     int32_t* tgt) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  tgt[i] = int32_t(splitmix64(hash3(seed, 103, uint64_t(row0 + i))) % uint64_t(V));
}

// One CTA-stride loop per row chunk: each thread writes 8 consecutive
// elements (one 16-byte vector) of both tensors.
__global__ void synth_logits_kernel(uint64_t seed, int64_t row0, int64_t rows, int32_t V,
                                    const int32_t* tgt, uint16_t* pol, uint16_t* ref) {
  const int64_t vec_per_row = V / 8;
  const int64_t total = rows * vec_per_row;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = g / vec_per_row;
    const int64_t v0 = (g - r * vec_per_row) * 8;
    const uint64_t rk = hash3(seed, 101, uint64_t(row0 + r));
    const int32_t y = tgt[r];
    uint32_t pw[4], qw[4];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const uint64_t h0 = splitmix64(rk + uint64_t(v0 + j));
      const uint64_t h1 = splitmix64(rk + uint64_t(v0 + j + 1));
      pw[j / 2] = uint32_t(synth_policy_bits(h0)) | (uint32_t(synth_policy_bits(h1)) << 16);
      qw[j / 2] = uint32_t(synth_ref_bits(h0, v0 + j == y)) |
                  (uint32_t(synth_ref_bits(h1, v0 + j + 1 == y)) << 16);
    }
    *reinterpret_cast<uint4*>(pol + r * int64_t(V) + v0) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
    *reinterpret_cast<uint4*>(ref + r * int64_t(V) + v0) = make_uint4(qw[0], qw[1], qw[2], qw[3]);
  }
}

__global__ void synth_floats_kernel(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n,
                                    int32_t kind, int32_t group_size, const float* base,
                                    float* out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t gi = uint64_t(i0 + i);
  const uint64_t key = hash3(seed, stream_id, gi);
  const uint64_t h = splitmix64(key);
  float v = 0.f;
  switch (kind) {
    case YATT_SYNTH_LOGP: v = -float(h >> 54) * (1.0f / 64.0f); break;
    case YATT_SYNTH_OLD_DELTA:
      v = (base ? base[i] : 0.f) + float(int(h >> 57) - 64) * (1.0f / 256.0f);
      break;
    case YATT_SYNTH_ADV: v = float(int(h >> 56) - 128) * (1.0f / 64.0f); break;
    case YATT_SYNTH_KL: v = float(h >> 56) * (1.0f / 1024.0f); break;
    case YATT_SYNTH_VALUE: v = float(int(h >> 53) - 1024) * (1.0f / 1024.0f); break;
    case YATT_SYNTH_REWARD: {
      const uint64_t g = gi / uint64_t(group_size);
      const uint64_t sel = splitmix64(hash3(seed, stream_id + 1000, g)) & 3;
      const double pg = sel == 0 ? 0.0
                        : sel == 1 ? 1.0
                        : sel == 2 ? 0.5
                                   : uniform_from_key(hash3(seed, stream_id + 2000, g));
      v = uniform_from_key(key) < pg ? 1.0f : 0.0f;
      break;
    }
    default: break;
  }
  out[i] = v;
}

}  // namespace

int synth_logits_launch(uint64_t seed, int64_t row0, int64_t rows, int32_t V, uint16_t* pol,
                        uint16_t* ref, int32_t* tgt, cudaStream_t st) {
  YATT_REQUIRE(V > 0 && V % 8 == 0, YATT_ERR_CONFIG, "synth_logits: vocab must be a multiple of 8");
  YATT_REQUIRE(rows >= 0, YATT_ERR_CONFIG, "synth_logits: rows must be >= 0");
  if (rows == 0) return YATT_OK;
  synth_targets_kernel<<<unsigned(ceil_div(rows, 256)), 256, 0, st>>>(seed, row0, rows, V, tgt);
  int rc = check_launch("synth_targets_kernel");
  if (rc) return rc;
  synth_logits_kernel<<<num_sms() * 8, 256, 0, st>>>(seed, row0, rows, V, tgt, pol, ref);
  return check_launch("synth_logits_kernel");
}

int synth_floats_launch(uint64_t seed, uint64_t stream_id, int64_t i0, int64_t n, int32_t kind,
                        int32_t group_size, const float* base, float* out, cudaStream_t st) {
  YATT_REQUIRE(kind >= YATT_SYNTH_LOGP && kind <= YATT_SYNTH_REWARD, YATT_ERR_CONFIG,
               "synth_floats: unknown kind %d", kind);
  YATT_REQUIRE(kind != YATT_SYNTH_REWARD || group_size > 0, YATT_ERR_CONFIG,
               "synth_floats: group_size must be positive for rewards");
  if (n <= 0) return YATT_OK;
  synth_floats_kernel<<<unsigned(ceil_div(n, 256)), 256, 0, st>>>(seed, stream_id, i0, n, kind,
                                                                   group_size, base, out);
  return check_launch("synth_floats_kernel");
}

}  // namespace yattb
