// frw_rng.cuh -- random streams of the B200 hot path.
//
//  * SplitMix64 parity streams: bit-identical to the reference generator
//    (proj/include/frwcap/rng.hpp:12-40), so a device transit/walk fed the
//    same (seed, stream) makes exactly the reference's decisions.
//  * Philox4x32-10 production streams (Salmon et al., SC'11): counter-based,
//    keyed by the 64-bit seed, counter = (transit/walk id, 32-bit step block,
//    domain word).  A draw is a pure function of (seed, id, step).
#pragma once
#include <cstdint>

namespace frw {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// state of SplitMix64(seed, stream) given mix(seed) (rng.hpp:16-17)
__host__ __device__ __forceinline__ uint64_t sm64_stream_from_mixed(
    uint64_t mixed_seed, uint64_t stream) {
  return sm64_mix(mixed_seed + (stream + 1) * kGamma);
}

// next() (rng.hpp:19-22)
__host__ __device__ __forceinline__ uint64_t sm64_next(uint64_t& s) {
  s += kGamma;
  return sm64_mix(s);
}

struct U32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U32x4 philox4x32_10(U32x4 c, uint32_t k0,
                                               uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = {hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

}  // namespace frw
