// Philox4x32-10 + Box-Muller on the device, bit-compatible with the
// reference generator (include/kvpack/rng.hpp:15-98): key = seed, counter =
// {block_lo, block_hi, stream_lo, stream_hi}; gaussian pair p comes from
// block p (u1 from words 0-1, u2 from words 2-3, 53-bit doubles), element 2p
// is r*cos(2*pi*u2) and element 2p+1 is r*sin(2*pi*u2).  Any element of a
// stream is computable independently, so whole matrices are generated in
// parallel (linalg.cpp:175-182 gaussian_matrix, harness.cpp:82-128).
#pragma once

#include <cstdint>

namespace kvp {

__host__ __device__ inline void philox10(uint32_t k0, uint32_t k1, uint32_t c[4]) {
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
    const uint64_t p2 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
    const uint32_t n0 = static_cast<uint32_t>(p2 >> 32) ^ c[1] ^ k0;
    const uint32_t n1 = static_cast<uint32_t>(p2);
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c[3] ^ k1;
    const uint32_t n3 = static_cast<uint32_t>(p0);
    c[0] = n0;
    c[1] = n1;
    c[2] = n2;
    c[3] = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Gaussian number `idx` of the stream (seed, stream), in double.
__host__ __device__ inline double philox_gaussian(uint64_t seed, uint64_t stream, uint64_t idx) {
  const uint64_t blk = idx >> 1;
  uint32_t c[4] = {static_cast<uint32_t>(blk), static_cast<uint32_t>(blk >> 32), static_cast<uint32_t>(stream),
                   static_cast<uint32_t>(stream >> 32)};
  philox10(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), c);
  double u1 = (static_cast<double>(c[0] >> 5) * 67108864.0 + static_cast<double>(c[1] >> 6)) * (1.0 / 9007199254740992.0);
  const double u2 = (static_cast<double>(c[2] >> 5) * 67108864.0 + static_cast<double>(c[3] >> 6)) * (1.0 / 9007199254740992.0);
  if (u1 <= 0.0) u1 = 1.0 / 9007199254740992.0;  // the reference redraws here (p = 2^-53)
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  return (idx & 1) ? r * sin(a) : r * cos(a);
}

// Philox stream ids of the synthetic harness (harness.cpp:29-32).
__host__ __device__ inline uint64_t stream_id(uint64_t purpose, uint64_t instance, uint64_t layer, uint64_t extra) {
  return (purpose << 56) | (instance << 24) | (layer << 8) | extra;
}

}  // namespace kvp
