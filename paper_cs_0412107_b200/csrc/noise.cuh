// noise.cuh -- device noise phi(c, k, i) of Eq. (4)/(5).
//
// One real N(0,1) per (chain c, sweep k, row i), shared by the z and w
// updates ("the noise term in (4) and in (5) are both the same"),
// never stored. Counter-based: Philox4x32-10 (Salmon et al., SC'11) with
// counter {i, k, c, 0} and key {seed lo, seed hi}, then the cosine branch of
// Box-Muller on two 53-bit uniforms (reading R4):
//   u1 = ((r0:r1 >> 11) + 1) 2^-53 in (0, 1],  u2 = (r2:r3 >> 11) 2^-53,
//   phi = sqrt(-2 ln u1) cos(2 pi u2).
#pragma once
#include <stdint.h>

namespace mcinv {

struct PhiloxOut {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ PhiloxOut philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   uint32_t k0, uint32_t k1) {
    constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
    constexpr uint32_t kWeyl0 = 0x9E3779B9u, kWeyl1 = 0xBB67AE85u;
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t hi0 = __umulhi(kMul0, c0), lo0 = kMul0 * c0;
        const uint32_t hi1 = __umulhi(kMul1, c2), lo1 = kMul1 * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += kWeyl0;
        k1 += kWeyl1;
    }
    return PhiloxOut{c0, c1, c2, c3};
}

__device__ __forceinline__ double box_muller(PhiloxOut r) {
    const unsigned long long a = (static_cast<unsigned long long>(r.x) << 32) | r.y;
    const unsigned long long b = (static_cast<unsigned long long>(r.z) << 32) | r.w;
    const double u1 = static_cast<double>((a >> 11) + 1ull) * 0x1p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__device__ __forceinline__ double gaussian(uint32_t row, uint32_t sweep, uint32_t chain, uint32_t k0,
                                           uint32_t k1) {
    return box_muller(philox4x32_10(row, sweep, chain, 0u, k0, k1));
}

}  // namespace mcinv
