// Philox4x32-10 counter-based RNG (Salmon et al., SC'11). Stateless: a draw is
// a pure function of (key, counter), so a head's draws are reproducible from
// (seed, epoch, worker, draw index) alone — this is what makes throughput
// mode resumable and independent of the launch geometry.
#pragma once
#include <stdint.h>

namespace nb {

struct u32x4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0,
                                                         uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
#else
    const uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

// Unbiased-enough bounded integer from 64 random bits (Lemire multiply-high;
// bias <= n / 2^64, the same order as the reference's rejection limit).
__host__ __device__ __forceinline__ uint32_t bounded(uint64_t r, uint32_t n) {
#ifdef __CUDA_ARCH__
  return (uint32_t)__umul64hi(r, (uint64_t)n);
#else
  return (uint32_t)(((unsigned __int128)r * n) >> 64);
#endif
}

__host__ __device__ __forceinline__ uint64_t join64(uint32_t hi, uint32_t lo) {
  return ((uint64_t)hi << 32) | lo;
}

}  // namespace nb
