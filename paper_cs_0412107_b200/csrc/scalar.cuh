// scalar.cuh -- real (double) / complex (cd) arithmetic used by the kernels.
//
// The complex fused multiply-add is defined componentwise (DESIGN.md reading
// R10):  re = fma(a.re, b.re, fma(-a.im, b.im, c.re)),
//        im = fma(a.re, b.im, fma( a.im, b.re, c.im)).
// The library is compiled with --fmad=false, so no other contraction occurs.
#pragma once
#include "mcinv_internal.cuh"

namespace mcinv {

template <typename S> struct ScalarTraits;
template <> struct ScalarTraits<double> { static constexpr int kDoubles = 1; };
template <> struct ScalarTraits<cd> { static constexpr int kDoubles = 2; };

template <typename S> __device__ __forceinline__ S zero_s();
template <> __device__ __forceinline__ double zero_s<double>() { return 0.0; }
template <> __device__ __forceinline__ cd zero_s<cd>() { return cd{0.0, 0.0}; }

__device__ __forceinline__ double fma_s(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ cd fma_s(cd a, cd b, cd c) {
    return cd{fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}

__device__ __forceinline__ double ldg_s(const double *p) { return __ldg(p); }
__device__ __forceinline__ cd ldg_s(const cd *p) {
    const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    return cd{v.x, v.y};
}

__device__ __forceinline__ double neg_s(double a) { return -a; }
__device__ __forceinline__ cd neg_s(cd a) { return cd{-a.re, -a.im}; }
__device__ __forceinline__ double conj_s(double a) { return a; }
__device__ __forceinline__ cd conj_s(cd a) { return cd{a.re, -a.im}; }
__device__ __forceinline__ double scale_s(double a, double x) { return a * x; }
__device__ __forceinline__ cd scale_s(cd a, double x) { return cd{a.re * x, a.im * x}; }
__device__ __forceinline__ double add_s(double a, double b) { return a + b; }
__device__ __forceinline__ cd add_s(cd a, cd b) { return cd{a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ double mul_s(double a, double b) { return a * b; }
__device__ __forceinline__ cd mul_s(cd a, cd b) { return cd{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
// z conj(w): the summand of Eq. (1/C)
__device__ __forceinline__ double zwc_s(double z, double w) { return z * w; }
__device__ __forceinline__ cd zwc_s(cd z, cd w) { return cd{z.re * w.re + z.im * w.im, z.im * w.re - z.re * w.im}; }

__device__ __forceinline__ double shfl_xor_s(double v, int off) { return __shfl_xor_sync(0xffffffffu, v, off); }
__device__ __forceinline__ cd shfl_xor_s(cd v, int off) {
    return cd{__shfl_xor_sync(0xffffffffu, v.re, off), __shfl_xor_sync(0xffffffffu, v.im, off)};
}

__device__ __forceinline__ void add_to(double *p, double v) { p[0] += v; }
__device__ __forceinline__ void add_to(double *p, cd v) { p[0] += v.re; p[1] += v.im; }

__device__ __forceinline__ void atomic_add_to(double *p, double v) { atomicAdd(p, v); }
__device__ __forceinline__ void atomic_add_to(double *p, cd v) {
    atomicAdd(p, v.re);
    atomicAdd(p + 1, v.im);
}

__device__ __forceinline__ bool bad_s(double v) { return !(fabs(v) <= 1e12); }
__device__ __forceinline__ bool bad_s(cd v) { return !(fabs(v.re) <= 1e12) || !(fabs(v.im) <= 1e12); }

}  // namespace mcinv
