// keyed_draw.cuh — sample_length_keyed (proj/src/workload.cpp:109-132,
// clamp_length :15-20, normal_from_key :23-27) on the device, with a
// certificate for the two distributions whose draw goes through libm.
//
// Constant / Uniform: IEEE multiply + nearbyint only — bit-identical to
// glibc by construction.
//
// Normal / LogNormal: the reference evaluates
//   z = sqrt(-2 * log1p(-u1)) * cos(2 pi u2),  v = p1 + p2 z  (or exp(v))
// with glibc.  Every operation here is rounded exactly like the reference's
// (the multiplies and the add are written as __dmul_rn / __dadd_rn, so no FMA
// contraction), except log1p, cos and exp, where CUDA's double routines and
// glibc's may differ by a couple of ulps (<= ~1e-15 relative after the
// composition).  The draw's integer length can therefore only differ from
// glibc's when v lies within that distance of a rounding boundary
// (x + 0.5; the clamp at 1 / max_len is applied after rounding and cannot
// flip a result).  The kernels flag every draw whose v lies within
// `band` * max(1, |v|) of a boundary (band default 1e-9: a 10^6x margin over
// the libm discrepancy); the host then redoes exactly those draws with
// glibc and re-runs with them as overrides (rollout_rounds.cu,
// yatt_sample_lengths_host).  The device value is used only where it is
// provably equal to glibc's.
#pragma once

#include <cmath>

#include "common.cuh"

namespace yattb {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kDefaultTieBand = 1e-9;

__host__ __device__ __forceinline__ int clamp_length(double value, int max_len) {
  const double rounded = nearbyint(value);
  if (rounded < 1) return 1;
  if (rounded > max_len) return max_len;
  return int(rounded);
}

__device__ __forceinline__ double normal_from_key_dev(uint64_t key) {
  const double u1 = uniform_from_key(key);
  const double u2 = uniform_from_key(splitmix64(key ^ 0x5bf0a8b1457e1d23ULL));
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log1p(-u1))), cos(__dmul_rn(kTwoPi, u2)));
}

// True when v is too close to a rounding boundary for the device value to be
// certified equal to glibc's.
__device__ __forceinline__ bool near_rounding_tie(double v, double band) {
  const double f = v - floor(v);  // exact
  return fabs(f - 0.5) <= band * fmax(1.0, fabs(v));
}

// Device draw.  *tie is set when the result is not certified (Normal /
// LogNormal only); the caller must then use the host (glibc) value.
__device__ __forceinline__ int length_keyed_dev(const yatt_length_dist& d, uint64_t seed,
                                                uint64_t stream, uint64_t step, uint64_t round,
                                                uint64_t id, double band, bool* tie) {
  *tie = false;
  const uint64_t key = hash5(seed, stream, step, round, id);
  switch (d.kind) {
    case YATT_DIST_CONSTANT: return clamp_length(d.p1, d.max_len_tokens);
    case YATT_DIST_UNIFORM: {
      const long long lo = llround(d.p1), hi = llround(d.p2);
      const uint64_t span = uint64_t(hi - lo) + 1;
      const double u = uniform_from_key(key);
      const long long v = lo + (long long)(__dmul_rn(u, double(span)));
      return clamp_length(double(v), d.max_len_tokens);
    }
    case YATT_DIST_NORMAL: {
      const double v = __dadd_rn(d.p1, __dmul_rn(d.p2, normal_from_key_dev(key)));
      *tie = near_rounding_tie(v, band);
      return clamp_length(v, d.max_len_tokens);
    }
    default: {
      const double v = exp(__dadd_rn(d.p1, __dmul_rn(d.p2, normal_from_key_dev(key))));
      *tie = near_rounding_tie(v, band);
      return clamp_length(v, d.max_len_tokens);
    }
  }
}

// Host draw with glibc — the reference's expression order exactly
// (workload.cpp:23-27, :109-132); host code, compiled by the host compiler.
int length_keyed_glibc(const yatt_length_dist& d, uint64_t seed, uint64_t stream, uint64_t step,
                       uint64_t round, uint64_t id);

// Certification band (tests widen it to force the host re-draw path).
double tie_band();

}  // namespace yattb
