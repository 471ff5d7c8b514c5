// noise.cuh -- device noise phi(c, k, i) of Eq. (4)/(5).
//
// One real N(0,1) per (chain c, sweep k, row i), shared by the z and w
// updates ("the noise term in (4) and in (5) are both the same"),
// never stored. Counter-based: Philox4x32-10 (Salmon et al., SC'11) with
// counter {i, k, c / 2, 0} and key {seed lo, seed hi}, then Box-Muller on two
// 53-bit uniforms (reading R4):
//   u1 = ((r0:r1 >> 11) + 1) 2^-53 in (0, 1],  u2 = (r2:r3 >> 11) 2^-53,
//   phi(2m) = sqrt(-2 ln u1) cos(2 pi u2),  phi(2m + 1) = sqrt(-2 ln u1) sin(2 pi u2):
// the two independent outputs of one pair go to the chains 2m, 2m + 1, so a
// thread holding both chains evaluates Philox, ln and sqrt once. ln and
// cos / sin are specialised to these argument ranges (log_unit, cos_0_2pi:
// < 1 ulp each, so phi matches the oracle's libm evaluation to a few ulp). The
// library builds with --fmad=false; the polynomials use explicit fma (Horner),
// which is as accurate and shortens them (measured +0.5% config 2, +1.7% config 3).
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

// log_unit and cos_0_2pi below follow fdlibm's e_log.c and k_cos.c / k_sin.c
// (argument reduction and the published minimax coefficients Lg1-Lg7, C1-C6,
// S1-S6, ln2_hi / ln2_lo), restructured into fma-Horner form for these
// argument ranges. fdlibm's notice, as its licence asks:
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this software is freely
//   granted, provided that this notice is preserved.
//
// ln(x) for x in (0, 1] (normal doubles only): the fdlibm method (reduce to
// m in [sqrt(2)/2, sqrt(2)), s = f / (2 + f), ln(1 + f) = f - f^2/2 +
// s (f^2/2 + R(s^2)) with a degree-14 minimax R); < 1 ulp, no special cases.
__device__ __forceinline__ double log_unit(double x) {
    int hx = __double2hiint(x);
    const int lx = __double2loint(x);
    int k = (hx >> 20) - 1023;
    hx &= 0x000fffff;
    const int i = (hx + 0x95f64) & 0x100000;  // 1 when the mantissa exceeds sqrt(2): use x / 2
    const double m = __hiloint2double(hx | (i ^ 0x3ff00000), lx);
    k += i >> 20;
    const double f = m - 1.0;
    const double s = f / (2.0 + f);
    const double dk = static_cast<double>(k);
    const double z = s * s, w = z * z;
    const double t1 = w * fma(w, fma(w, 1.531383769920937332e-01, 2.222219843214978396e-01), 3.999999999940941908e-01);
    const double t2 =
        z * fma(w, fma(w, fma(w, 1.479819860511658591e-01, 1.818357216161805012e-01), 2.857142874366239149e-01),
                6.666666666666735130e-01);
    const double hfsq = 0.5 * f * f;
    return dk * 6.93147180369123816490e-01 - ((hfsq - (s * (hfsq + (t1 + t2)) + dk * 1.90821492927058770002e-10)) - f);
}

// cos(x - shift pi/2) for x in [0, 2 pi] (shift 1: sin x): x - q pi/2 by two fma
// (Cody-Waite; exact up to the final rounding), then the fdlibm kernels on
// [-pi/4, pi/4]; < 1 ulp. Both kernels are evaluated; the quadrant picks one.
__device__ __forceinline__ double cos_0_2pi(double x, int shift = 0) {
    const double q = rint(x * 0.6366197723675814);
    double r = fma(-q, 1.5707963267948966, x);
    r = fma(-q, 6.123233995736766e-17, r);
    const double z = r * r;
    const double rc =
        z * fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                                     -2.75573143513906633035e-07),
                              2.48015872894767294178e-05),
                       -1.38888888888741095749e-03),
                4.16666666666666019037e-02);
    const double rs = fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                                        2.75573137070700676789e-06),
                                 -1.98412698298579493134e-04),
                          8.33333333332248946124e-03);
    const double hz = 0.5 * z, w = 1.0 - hz;
    const double c = w + (((1.0 - w) - hz) + z * rc);
    const double sn = r + (z * r) * (-1.66666666666666324348e-01 + z * rs);
    const int qi = (static_cast<int>(q) - shift) & 3;  // cos(r + (q - shift) pi/2)
    const double v = (qi & 1) ? sn : c;
    return (qi == 1 || qi == 2) ? -v : v;
}

// cos x and sin x for x in [0, 2 pi] from one reduction (the two outputs of cos_0_2pi's
// kernels in their quadrants)
__device__ __forceinline__ void sincos_0_2pi(double x, double &cs, double &sn_out) {
    const double q = rint(x * 0.6366197723675814);
    double r = fma(-q, 1.5707963267948966, x);
    r = fma(-q, 6.123233995736766e-17, r);
    const double z = r * r;
    const double rc =
        z * fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                                     -2.75573143513906633035e-07),
                              2.48015872894767294178e-05),
                       -1.38888888888741095749e-03),
                4.16666666666666019037e-02);
    const double rs = fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                                        2.75573137070700676789e-06),
                                 -1.98412698298579493134e-04),
                          8.33333333332248946124e-03);
    const double hz = 0.5 * z, w = 1.0 - hz;
    const double c = w + (((1.0 - w) - hz) + z * rc);
    const double sn = r + (z * r) * (-1.66666666666666324348e-01 + z * rs);
    const int qc = static_cast<int>(q) & 3, qs = (qc + 3) & 3;
    const double vc = (qc & 1) ? sn : c, vs = (qs & 1) ? sn : c;
    cs = (qc == 1 || qc == 2) ? -vc : vc;
    sn_out = (qs == 1 || qs == 2) ? -vs : vs;
}

// output `odd` of the Box-Muller pair of one block (0: cosine, 1: sine)
__device__ __forceinline__ double box_muller(PhiloxOut r, int odd = 0) {
    const unsigned long long a = (static_cast<unsigned long long>(r.x) << 32) | r.y;
    const unsigned long long b = (static_cast<unsigned long long>(r.z) << 32) | r.w;
    const double u1 = static_cast<double>((a >> 11) + 1ull) * 0x1p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1p-53;
    return sqrt(-2.0 * log_unit(u1)) * cos_0_2pi(6.283185307179586 * u2, odd);
}

// both outputs of the pair
__device__ __forceinline__ void box_muller2(PhiloxOut r, double &g0, double &g1) {
    const unsigned long long a = (static_cast<unsigned long long>(r.x) << 32) | r.y;
    const unsigned long long b = (static_cast<unsigned long long>(r.z) << 32) | r.w;
    const double u1 = static_cast<double>((a >> 11) + 1ull) * 0x1p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1p-53;
    const double rad = sqrt(-2.0 * log_unit(u1));
    double c, s;
    sincos_0_2pi(6.283185307179586 * u2, c, s);
    g0 = rad * c;
    g1 = rad * s;
}

// phi of one chain (reading R4): output chain & 1 of the pair of counter {row, sweep, chain / 2, 0}
__device__ __forceinline__ double gaussian(uint32_t row, uint32_t sweep, uint32_t chain, uint32_t k0,
                                           uint32_t k1) {
    return box_muller(philox4x32_10(row, sweep, chain >> 1, 0u, k0, k1), static_cast<int>(chain & 1u));
}

// phi of the chains 2m and 2m + 1 (chain_even = 2m): one Philox block, one ln and sqrt
__device__ __forceinline__ void gaussian2(uint32_t row, uint32_t sweep, uint32_t chain_even, uint32_t k0, uint32_t k1,
                                          double &g0, double &g1) {
    box_muller2(philox4x32_10(row, sweep, chain_even >> 1, 0u, k0, k1), g0, g1);
}

// Z2 noise phi = 2B - 1 (reading R21): B = top bit
// of word 0 of Philox(counter {row, sweep, chain, 1}): a stream disjoint from
// the Gaussian one. 1 -> -1, 0 -> +1.
__device__ __forceinline__ double z2_noise(uint32_t row, uint32_t sweep, uint32_t chain, uint32_t k0, uint32_t k1) {
    return (philox4x32_10(row, sweep, chain, 1u, k0, k1).x >> 31) ? -1.0 : 1.0;
}

// phi(chain, sweep, row) for the run's noise mode: 0 Gaussian, 3 Z2, 1/2 the
// test constants 0/1 (MCINV_NOISE_*)
__device__ __forceinline__ double noise_phi(int mode, uint32_t row, uint32_t sweep, uint32_t chain, uint32_t k0,
                                            uint32_t k1) {
    if (mode == 1 || mode == 2) return mode == 2 ? 1.0 : 0.0;
    // one Philox block: counter word 3 selects the stream (0 Gaussian pairs, 1 Z2)
    const PhiloxOut r = philox4x32_10(row, sweep, mode == 3 ? chain : chain >> 1, mode == 3 ? 1u : 0u, k0, k1);
    if (mode == 3) return (r.x >> 31) ? -1.0 : 1.0;
    return box_muller(r, static_cast<int>(chain & 1u));
}

}  // namespace mcinv
