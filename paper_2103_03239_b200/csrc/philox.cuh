// philox.cuh -- counter-based Philox4x32-10 normals (Salmon et al., SC'11)
// for the device-noise Moshpit SGD path.  Counter (step, peer, quad of 4
// coordinates), key = seed: the fused and unfused kernels draw identical
// noise for the same (step, peer, coordinate).
#pragma once
#include <cstdint>

namespace mb200 {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const std::uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// Four standard normals for (step, peer, quad) via Box-Muller in fp32 (full-
// rate SFU math; the device-noise path promises statistical parity only).
__device__ __forceinline__ void philox_normals4(std::uint64_t seed, std::uint64_t step,
                                                std::uint64_t peer, std::uint64_t quad,
                                                double z[4]) {
  const uint4 r = philox4x32_10(
      make_uint4((std::uint32_t)step, (std::uint32_t)peer, (std::uint32_t)quad,
                 (std::uint32_t)(quad >> 32)),
      make_uint2((std::uint32_t)seed, (std::uint32_t)(seed >> 32)));
  const std::uint32_t a[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    // u1 in (0, 1]: top 24 bits + 1 ulp, exact in fp32
    const float u1 = (float)((a[2 * h] >> 8) + 1u) * 0x1.0p-24f;
    const float u2 = (float)(a[2 * h + 1] >> 8) * 0x1.0p-24f;
    const float rr = sqrtf(-2.0f * logf(u1));
    float s, c;
    sincospif(2.0f * u2, &s, &c);
    z[2 * h] = (double)(rr * c);
    z[2 * h + 1] = (double)(rr * s);
  }
}

}  // namespace mb200
