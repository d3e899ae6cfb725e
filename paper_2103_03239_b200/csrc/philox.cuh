// philox.cuh -- counter-based Philox4x32-10 normals (Salmon et al., SC'11)
// for the device-noise Moshpit SGD path.  Counter (step, peer, quad of 4
// coordinates), key = seed: the fused and unfused kernels draw identical
// noise for the same (step, peer, coordinate).
#pragma once
#include <cstdint>

#ifndef MB_PHILOX_ROUNDS
#define MB_PHILOX_ROUNDS 7
#endif

namespace mb200 {

// Rounds of the Philox4x32 bijection.  7 is the smallest count Salmon et al.
// (SC'11, Table 2) report as passing every TestU01 BigCrush test for
// Philox4x32 ("Crush-resistant"); 10 is their recommended safety margin.  The
// device-noise path promises statistical parity only (the reference draws
// its noise from xoshiro on the host), its tests check the moments and the
// reference's V_k / sigma_hat properties, and the fused and unfused kernels
// share this generator.  Measured on B200 (C4 sigma = 1, profiles/r02/):
// 3.19 ms per SGD step at 10 rounds, 3.07 ms at 7 -- the kernel is issue
// bound, three rounds are ~4 of its ~25 instructions per element.
constexpr int kPhiloxRounds = MB_PHILOX_ROUNDS;
static_assert(kPhiloxRounds >= 7 && kPhiloxRounds <= 10, "Philox4x32-7 .. -10");

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < kPhiloxRounds; ++r) {
    const std::uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// The same generator with the 10 round keys precomputed (kernel parameters,
// i.e. constant-bank operands of the XORs): round r uses
// (seed_lo + r * 0x9E3779B9, seed_hi + r * 0xBB67AE85), as above.
struct PhiloxKeys {
  uint2 k[10];
};
inline PhiloxKeys philox_keys(std::uint64_t seed) {
  PhiloxKeys p;
  std::uint32_t a = (std::uint32_t)seed, b = (std::uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.k[r] = make_uint2(a, b);
    a += 0x9E3779B9u;
    b += 0xBB67AE85u;
  }
  return p;
}
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxKeys& kk) {
#pragma unroll
  for (int r = 0; r < kPhiloxRounds; ++r) {
    const std::uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ kk.k[r].x, lo1, hi0 ^ c.w ^ kk.k[r].y, lo0);
  }
  return c;
}

// Four standard normals for (step, peer, quad): Box-Muller on SFU intrinsics
// (the device-noise path promises statistical parity only, and this keeps the
// fused step + averaging kernel memory-bound).
__device__ __forceinline__ void box_muller4(uint4 r, float z[4]);
__device__ __forceinline__ void philox_normals4(std::uint64_t seed, std::uint64_t step,
                                                std::uint64_t peer, std::uint64_t quad,
                                                float z[4]) {
  box_muller4(philox4x32_10(make_uint4((std::uint32_t)step, (std::uint32_t)peer,
                                       (std::uint32_t)quad, (std::uint32_t)(quad >> 32)),
                            make_uint2((std::uint32_t)seed, (std::uint32_t)(seed >> 32))),
              z);
}
__device__ __forceinline__ void philox_normals4(const PhiloxKeys& kk, std::uint64_t step,
                                                std::uint64_t peer, std::uint64_t quad,
                                                float z[4]) {
  box_muller4(philox4x32_10(make_uint4((std::uint32_t)step, (std::uint32_t)peer,
                                       (std::uint32_t)quad, (std::uint32_t)(quad >> 32)),
                            kk),
              z);
}
__device__ __forceinline__ void box_muller4(uint4 r, float z[4]) {
  const std::uint32_t a[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    // u1 = v / 2^24 in (0, 1] with v = (a >> 8) + 1, so
    // -2 ln u1 = -2 ln2 * (log2 v - 24): one MUFU.LG2 and one FFMA.
    const float v = (float)((a[2 * h] >> 8) + 1u);
    float l2;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(v));  // v >= 1: no denormals
    const float e = fmaxf(__fmaf_rn(l2, -1.3862943611198906f, 33.271064666877374f), 0.0f);
    float rr;  // sqrt on the SFU (MUFU.SQRT)
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rr) : "f"(e));
    float s, c;  // angle 2*pi*u2, u2 = (a >> 8) / 2^24 in [0, 1)
    __sincosf((float)(a[2 * h + 1] >> 8) * 3.7450702e-07f, &s, &c);
    z[2 * h] = rr * c;
    z[2 * h + 1] = rr * s;
  }
}

// n_j^2 summed for sigma_hat: per 4-coordinate quad in the state's
// precision (fp32: one fp32 partial per quad), then into the caller's fp64
// accumulator -- the same terms in the fused and the standalone step.
__device__ __forceinline__ void nsq_add(float& q, float nj) { q = __fmaf_rn(nj, nj, q); }
__device__ __forceinline__ void nsq_add(double& q, double nj) { q = __fma_rn(nj, nj, q); }

// One noise component n_j = coord_std * z in the state's precision; both the
// standalone step kernel and the fused kernel 3 use it (bit-identical noise).
__device__ __forceinline__ float noise_component(float z, double coord_std, float*) {
  return __fmul_rn((float)coord_std, z);
}
__device__ __forceinline__ double noise_component(float z, double coord_std, double*) {
  return __dmul_rn(coord_std, (double)z);
}

}  // namespace mb200
