// contract_ozaki.cu -- K3 (alternative, MCINV_CONTRACT_OZAKI=1): the full-inverse accumulation
// A_g += X_g Y_g^dagger (Eq. 1/C) as FP64 by the Ozaki scheme on the 5th-generation
// tensor cores' INT8 path (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Each row i of X_g (its K = T * gs samples of one SE group, real and imaginary parts) is scaled
// by a power of two 2^-e_i so that its entries lie in (-1, 1) and split exactly into NS signed
// 7-bit digits (int8 "slices"): x = 2^e_i sum_s a_s 2^-7(s+1) + residual, |residual| < 2^(e_i - 7 NS).
// Y likewise with f_j. Then
//     X Y^T = sum_{s+t < NS} 2^(e_i + f_j - 7(s+t+2)) (A_s B_t^T)
// where every A_s B_t^T is an int8 GEMM with exact int32 accumulation; the products of one level
// L = s + t share a TMEM accumulator (at most NS * K' * 127^2 < 2^31), and the epilogue converts
// the NS levels to fp64, scales them and adds them into A_g. Complex: Re = [Xr | Xi] [Yr | Yi]^T,
// Im = [Xi | -Xr] [Yr | Yi]^T, two passes over K' = 2K. The dropped terms are below 2^-7NS of
// the row/column scales (NS = 6: 2^-42 ~ 2e-13).
//
// GEMM tile 128 x 64 (one TMEM accumulator of 64 columns per level), K staged in chunks of 64 int8
// per slice by TMA (64-B swizzle, K-major), all NS slices of both operands per stage, a ring of KS
// stages. The B slice tiles are stacked in shared memory, so A_s B_t^T for up to four consecutive t
// is ONE MMA (UMMA M = 128, N = 64 m <= 256, K = 32) writing the consecutive level accumulators
// s + t: 8 MMAs per K step instead of 21 N = 64 ones (an N = 64 MMA is bound by shared-memory
// reads of its A tile; measured 51 vs 32 compute cycles, tools/micro/umma_bench.cu).
// One thread streams the stages (bulk copies of the pre-swizzled digit tiles), another issues the
// MMAs; tcgen05.commit frees a stage; eight warps read the NS accumulators (tcgen05.ld) in the
// epilogue, combine them exactly in int64 and add the tile into A_g.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "mcinv_internal.cuh"
#include "scalar.cuh"

namespace mcinv {
namespace {

#ifndef MCINV_OZ_KC
#define MCINV_OZ_KC 64  // K chunk per stage (bytes of one row): 64 (64-B swizzle) or 32 (32-B swizzle)
#endif
constexpr int OZ_M = 128, OZ_N = 64, OZ_KC = MCINV_OZ_KC;  // tile and K chunk (int8 = bytes)
constexpr int OZ_KS = OZ_KC == 64 ? 3 : 6;                   // stages (216 KB of shared memory)

__device__ __forceinline__ uint32_t s_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- slicing
// One CTA per row of one operand of one SE group: the row's K samples (snapshot sweep t,
// chain c of group g: k = t gs + c) -> exponent and NS int8 digits per part.
// X: A[s][i][k'] = digit of [Xr | Xi], A2[s][i][k'] = digit of [Xi | -Xr];  Y: B[s][j][k'] of [Yr | Yi].
// Real: A[s][i][k] of X (K' = K), no A2. Columns k' >= K' (padding to the K chunk) are zero.
//
// Digit layout (P = panel height: 128 for X, 64 for Y; rows padded to a multiple of P with zeros):
// tiled (default) -- the bytes one pipeline stage of one GEMM tile needs are contiguous in global
// memory: [panel][K chunk of 64][slice][row in panel][64 bytes], each 8-row x 64-B atom already in
// the 64-B swizzle UMMA reads (16-B unit u of row r stored at u ^ ((r >> 1) & 3)), so a stage is
// two linear bulk copies; plain (MCINV_OZ_BULK=0) -- [slice][row][k'] fetched by tensor-map TMA.
__device__ __forceinline__ size_t digit_at(bool tiled, int P, int nk, int NS, size_t plane, int Kp, int s, int row,
                                           int k) {
    if (!tiled) return s * plane + (size_t)row * Kp + k;
    const int p = row / P, rr = row - p * P, kc = k >> 6, kb = k & 63;
    return ((((size_t)p * nk + kc) * NS + s) * P + rr) * 64 + ((((kb >> 4) ^ ((rr >> 1) & 3)) << 4) | (kb & 15));
}

template <typename S, int NS>
__global__ void ozaki_slice_kernel(const S *__restrict__ snap, int n, int ld, int gs, int g, int K, int Kp,
                                   int8_t *__restrict__ out, int8_t *__restrict__ out2, int *__restrict__ expo,
                                   int tiled, int P) {
    constexpr bool CPLX = ScalarTraits<S>::kDoubles == 2;
    const int i = blockIdx.x;  // rows i >= n (tiled padding) write zero digits
    const int nk = Kp >> 6;
    __shared__ double red[32];
    double mx = 0.0;
    for (int k = threadIdx.x; k < K && i < n; k += blockDim.x) {
        const int t = k / gs, c = k - t * gs;
        const S v = snap[((int64_t)t * n + i) * ld + (int64_t)g * gs + c];
        if constexpr (CPLX) mx = fmax(mx, fmax(fabs(v.re), fabs(v.im)));
        else mx = fmax(mx, fabs(v));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    int e = 0;
    if (red[0] > 0.0) frexp(red[0], &e);  // max in [2^(e-1), 2^e): scaled entries in (-1, 1)
    if (threadIdx.x == 0 && i < n) expo[i] = e;
    const size_t plane = (size_t)n * Kp;
    auto at = [&](int s, int k) { return digit_at(tiled != 0, P, nk, NS, plane, Kp, s, i, k); };
    auto digits = [&](double x, int8_t (&d)[NS]) {
        double r = ldexp(x, -e);  // exact
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            r *= 128.0;  // exact
            const double q = trunc(r);
            d[s] = static_cast<int8_t>(q);
            r -= q;  // exact
        }
    };
    for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
        int8_t d0[NS], d1[NS];
        if (k < K && i < n) {
            const int t = k / gs, c = k - t * gs;
            const S v = snap[((int64_t)t * n + i) * ld + (int64_t)g * gs + c];
            if constexpr (CPLX) {
                digits(v.re, d0);
                digits(v.im, d1);
            } else {
                digits(v, d0);
            }
        } else {
#pragma unroll
            for (int s = 0; s < NS; ++s) d0[s] = d1[s] = 0;
        }
        if constexpr (CPLX) {
            const int Kh = Kp / 2;  // the K' layout is [re part | im part], each padded to Kh
            if (k < Kh) {
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    out[at(s, k)] = d0[s];
                    out[at(s, Kh + k)] = d1[s];
                    if (out2) {
                        out2[at(s, k)] = d1[s];
                        out2[at(s, Kh + k)] = static_cast<int8_t>(-d0[s]);
                    }
                }
            }
        } else {
#pragma unroll
            for (int s = 0; s < NS; ++s) out[at(s, k)] = d0[s];
        }
    }
}

// The same digits written in the tiled layout 8 k' at a time: each thread keeps 8 scaled values in
// registers and stores 8 bytes (half a swizzle unit) per slice and part, instead of byte stores.
template <typename S, int NS>
__global__ void __launch_bounds__(128, 6) ozaki_slice_tiled_kernel(const S *__restrict__ snap, int n, int ld, int gs, int g0,
                                                            int K, int Kp, int8_t *__restrict__ out,
                                                            int8_t *__restrict__ out2, int *__restrict__ expo, int P,
                                                            size_t slot) {
    constexpr bool CPLX = ScalarTraits<S>::kDoubles == 2;
    // a batch of SE groups: blockIdx.x = group in the batch (the CTAs of one row read neighbouring
    // columns of the snapshots), blockIdx.y = row; group b's digits live in scratch slot b
    const int g = g0 + blockIdx.x, i = blockIdx.y;  // rows i >= n (panel padding) write zero digits
    out += blockIdx.x * slot;
    if (out2) out2 += blockIdx.x * slot;
    expo = reinterpret_cast<int *>(reinterpret_cast<char *>(expo) + blockIdx.x * slot);
    __shared__ double red[32];
    double mx = 0.0;
    for (int k = threadIdx.x; k < K && i < n; k += blockDim.x) {
        const int t = k / gs, c = k - t * gs;
        const S v = snap[((int64_t)t * n + i) * ld + (int64_t)g * gs + c];
        if constexpr (CPLX) mx = fmax(mx, fmax(fabs(v.re), fabs(v.im)));
        else mx = fmax(mx, fabs(v));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    int e = 0;
    if (red[0] > 0.0) frexp(red[0], &e);  // max in [2^(e-1), 2^e): scaled entries in (-1, 1)
    if (threadIdx.x == 0 && i < n) expo[i] = e;
    const int nk = Kp >> 6, p = i / P, rr = i - p * P, sw = (rr >> 1) & 3;
    // the 8 bytes holding k' = k..k+7 (k % 8 == 0): half (k >> 3) & 1 of 16-byte unit (k >> 4) & 3
    auto half_unit = [&](int8_t *o, int s, int k) {
        return reinterpret_cast<uint2 *>(o + ((((size_t)p * nk + (k >> 6)) * NS + s) * P + rr) * 64 +
                                         ((((k >> 4) & 3) ^ sw) << 4) + (((k >> 3) & 1) << 3));
    };
    // x 2^-e as a multiplication when 2^-e is a normal double: exactly ldexp(x, -e)
    const bool mul_ok = e > -1022 && e < 1022;
    const double sc = mul_ok ? __longlong_as_double((long long)(1023 - e) << 52) : 1.0;
    const int KU = CPLX ? Kp / 2 : Kp;  // complex: k' = [re part | im part], each KU wide
    // segments of 8 x 128 samples: coalesced loads into shared memory (one 8-sample group per
    // thread, padded by one element per group so a warp's 16-byte reads spread over the banks)
    constexpr int SEG = 8 * 128;
    __shared__ S seg[SEG + SEG / 8];
    for (int s0 = 0; s0 < KU; s0 += SEG) {
        __syncthreads();
        for (int k = s0 + threadIdx.x; k < s0 + SEG; k += blockDim.x) {
            S v{};
            if (k < K && i < n) {
                const int t = k / gs, c = k - t * gs;
                v = snap[((int64_t)t * n + i) * ld + (int64_t)g * gs + c];
            }
            seg[(k - s0) + (k - s0) / 8] = v;
        }
        __syncthreads();
        const int k0 = s0 + threadIdx.x * 8;
        if (k0 >= KU) continue;
        double a[8], b[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const S v = seg[threadIdx.x * 9 + j];
            if constexpr (CPLX) {
                a[j] = mul_ok ? v.re * sc : ldexp(v.re, -e);  // exact
                b[j] = mul_ok ? v.im * sc : ldexp(v.im, -e);
            } else {
                a[j] = mul_ok ? v * sc : ldexp(v, -e);
                b[j] = 0.0;
            }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            uint32_t pa[2] = {0, 0}, pb[2] = {0, 0}, na[2] = {0, 0};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                a[j] *= 128.0;  // exact
                const double qa = trunc(a[j]);
                a[j] -= qa;  // exact
                const int da = static_cast<int>(qa);
                pa[j >> 2] |= (uint32_t)(uint8_t)(int8_t)da << (8 * (j & 3));
                na[j >> 2] |= (uint32_t)(uint8_t)(int8_t)(-da) << (8 * (j & 3));
                if constexpr (CPLX) {
                    b[j] *= 128.0;
                    const double qb = trunc(b[j]);
                    b[j] -= qb;
                    pb[j >> 2] |= (uint32_t)(uint8_t)(int8_t) static_cast<int>(qb) << (8 * (j & 3));
                }
            }
            *half_unit(out, s, k0) = make_uint2(pa[0], pa[1]);
            if constexpr (CPLX) {
                *half_unit(out, s, KU + k0) = make_uint2(pb[0], pb[1]);
                if (out2) {
                    *half_unit(out2, s, k0) = make_uint2(pb[0], pb[1]);
                    *half_unit(out2, s, KU + k0) = make_uint2(na[0], na[1]);
                }
            }
        }
    }
}

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_waitp(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred q;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, q;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// linear bulk copy global -> shared (the tiled digit layout), completion on the stage's mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
#ifdef MCINV_OZ_PROF  // cycle buckets summed over CTAs: [wait full, issue MMAs] of the MMA thread,
                      // [wait empty, issue copies] of the producer, then per-CTA phases
__device__ unsigned long long g_oz_prof[12];
#define OZ_P(k)                                     \
    do {                                            \
        if (threadIdx.x == 0) ph_[(k)] = clock64(); \
    } while (0)
#define OZ_CLK(v) const long long v = clock64()
#define OZ_ADD(b, a, z) prof_[(b)] += (z) - (a)
#else
#define OZ_P(k) \
    do {        \
    } while (0)
#define OZ_CLK(v) \
    do {          \
    } while (0)
#define OZ_ADD(b, a, z) \
    do {                \
    } while (0)
#endif
// shared-memory matrix descriptor, K-major, 64-B swizzle: rows of 64 B, 8-row groups 512 B apart
// (SBO = 32 x 16 B), LBO = 1 (unused by swizzled K-major), version 1 (sm_100), layout 4 = SWIZZLE_64B
// (KC = 32: rows of 32 B, 8-row groups 256 B apart, layout 6 = SWIZZLE_32B)
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(OZ_KC == 64 ? 32 : 16) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(OZ_KC == 64 ? 4 : 6) << 61;
    return d;
}
// instruction descriptor: s8 x s8 -> s32, K-major A and B, M = 128, N = nn (a multiple of 64 here, <= 256)
__host__ __device__ constexpr uint32_t idesc_i8(int nn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nn >> 3) << 17) | ((uint32_t)(OZ_M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    const uint32_t mask0 = 0, mask1 = 0, mask2 = 0, mask3 = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(mask0), "r"(mask1), "r"(mask2), "r"(mask3));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// ---------------------------------------------------------------- GEMM + epilogue
// 16 columns (block q) of the tile's value sum_L 2^(x - 7(L+2)) D_L, x = e_i + f_j, for this
// thread's TMEM lane: levels 0-2 and 3-5 combine exactly in int64 (hi = (D0 2^7 + D1) 2^7 + D2 <
// 2^46, lo likewise), so each element is fma(lo, 2^(x-49), hi 2^(x-28)): one rounding.
template <int NS>
__device__ __forceinline__ void level_values16(uint32_t lane_addr, int q, int ei, const int *eys, double (&v)[16]) {
    static_assert(NS == 6, "the epilogue groups the levels 3 + 3");
    uint32_t d[NS][16];
#pragma unroll
    for (int L = 0; L < NS; ++L)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(d[L][0]), "=r"(d[L][1]), "=r"(d[L][2]), "=r"(d[L][3]), "=r"(d[L][4]), "=r"(d[L][5]),
              "=r"(d[L][6]), "=r"(d[L][7]), "=r"(d[L][8]), "=r"(d[L][9]), "=r"(d[L][10]), "=r"(d[L][11]),
              "=r"(d[L][12]), "=r"(d[L][13]), "=r"(d[L][14]), "=r"(d[L][15])
            : "r"(lane_addr + (uint32_t)(L * OZ_N + q * 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        long long hi = 0, lo = 0;
#pragma unroll
        for (int L = 0; L < 3; ++L) {
            hi = hi * 128 + static_cast<int32_t>(d[L][c]);
            lo = lo * 128 + static_cast<int32_t>(d[L + 3][c]);
        }
        const int x = ei + eys[q * 16 + c];
        if (x > -960 && x < 1000)  // 2^(x-28) and 2^(x-49) are normal doubles
            v[c] = fma(static_cast<double>(lo), __longlong_as_double((long long)(x - 49 + 1023) << 52),
                       static_cast<double>(hi) * __longlong_as_double((long long)(x - 28 + 1023) << 52));
        else
            v[c] = ldexp(fma(static_cast<double>(lo), 0x1p-21, static_cast<double>(hi)), x - 28);
    }
}

// TMEM columns 384..511 (free: the NS = 6 levels use 0..383) hold the real part of a complex tile
// as fp64 (two 32-bit columns per element) while the imaginary part's MMAs reuse the accumulators
constexpr int kReCol = 6 * 64;
__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
}

// out: A_g (fp64, e doubles per element): out[(i n + j) e + part] += sum_L 2^(ei + fj - 7(L+2)) D_L[i][j].
// FUSED (complex, tiled digits): phase 0 contracts A = [Xr | Xi] (real part), phase 1 A2 = [Xi | -Xr]
// (imaginary part) against the same B in one CTA: the real tile is parked in TMEM between them, and
// one epilogue adds whole complex elements (16-byte accesses) into A_g.
template <int NS, bool BULK, bool FUSED>
__global__ void __launch_bounds__(256, 1) ozaki_gemm_kernel(const __grid_constant__ CUtensorMap ma,
                                                            const __grid_constant__ CUtensorMap mb,
                                                            const int8_t *__restrict__ ga, const int8_t *__restrict__ ga2,
                                                            const int8_t *__restrict__ gb,
                                                            const int *__restrict__ ex, const int *__restrict__ ey,
                                                            double *__restrict__ out, int n, int e, int part, int Kp) {
    static_assert(!FUSED || BULK, "the fused complex kernel reads the tiled digits");
    constexpr int PH = FUSED ? 2 : 1;
    constexpr uint32_t kA = OZ_M * OZ_KC, kB = OZ_N * OZ_KC;  // bytes of one slice tile
    constexpr uint32_t kStage = NS * (kA + kB);
    extern __shared__ __align__(128) unsigned char smo[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smo) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = s_addr(base);
    // after the ring: full[KS], empty[KS], done, re_full (phase 0 accumulated), re_free (real part
    // parked, accumulators free), the TMEM address, f_j of the tile's columns
    const uint32_t full = sbase + OZ_KS * kStage, empty = full + 8 * OZ_KS, done = empty + 8 * OZ_KS;
    const uint32_t re_full = done + 8, re_free = done + 16;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(base + OZ_KS * kStage + 16 * OZ_KS + 24);
    int *eys = reinterpret_cast<int *>(base + OZ_KS * kStage + 16 * OZ_KS + 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef MCINV_OZ_PROF
    long long ph_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, prof_[4] = {0, 0, 0, 0};
#endif
    OZ_P(0);
    const int i0 = blockIdx.y * OZ_M, j0 = blockIdx.x * OZ_N;
    const int nk = Kp / OZ_KC;
    if (threadIdx.x == 0) {
        for (int q = 0; q < OZ_KS; ++q) {
            mbar_init1(full + 8 * q);
            mbar_init1(empty + 8 * q);
        }
        mbar_init1(done);
        mbar_init1(re_full);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(re_free) : "memory");  // one arrival per warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // 512 TMEM columns: NS accumulators of N = 64 int32 columns (+ the parked real part)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x < OZ_N) eys[threadIdx.x] = j0 + (int)threadIdx.x < n ? ey[j0 + threadIdx.x] : 0;
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(tmem_slot);
    const int lq = warp & 3, ch = warp >> 2;  // TMEM lane quarter (warp % 4 by hardware), column half
    const int r = lq * 32 + lane, i = i0 + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(lq * 32) << 16);
    const int ei = i < n ? ex[i] : 0;

    // warp specialisation: warp 1 lane 0 streams the stages (producer), warp 0 lane 0 issues the
    // MMAs; warps 4-7 park the real part (FUSED); all eight warps run the final epilogue
    if (warp == 1 && lane == 0) {
        for (int it = 0; it < PH * nk; ++it) {
            const int ph = it >= nk, kc = it - ph * nk, q = it % OZ_KS;
            const uint32_t st = sbase + q * kStage;
            OZ_CLK(ta);
            if (it >= OZ_KS) mbar_waitp(empty + 8 * q, (uint32_t)(((it / OZ_KS) - 1) & 1));  // chunk it - KS done
            OZ_CLK(tb);
            mbar_expect(full + 8 * q, kStage);
            if constexpr (BULK) {  // [panel][chunk][slice][row][64]: one stage of A, one of B
                bulk_g2s(st, (ph ? ga2 : ga) + ((size_t)blockIdx.y * nk + kc) * (NS * kA), NS * kA, full + 8 * q);
                bulk_g2s(st + NS * kA, gb + ((size_t)blockIdx.x * nk + kc) * (NS * kB), NS * kB, full + 8 * q);
            } else {
                for (int s = 0; s < NS; ++s) {
                    tma3(st + s * kA, &ma, kc * OZ_KC, i0, s, full + 8 * q);
                    tma3(st + NS * kA + s * kB, &mb, kc * OZ_KC, j0, s, full + 8 * q);
                }
            }
            OZ_CLK(tc);
            OZ_ADD(2, ta, tb);
            OZ_ADD(3, tb, tc);
        }
    } else if (threadIdx.x == 0) {
        OZ_P(1);
        for (int it = 0; it < PH * nk; ++it) {
            const int ph = it >= nk, kc = it - ph * nk, q = it % OZ_KS;
            if (FUSED && ph == 1 && kc == 0) {  // the real part must be parked before its columns are reused
                mbar_waitp(re_free, 0);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            OZ_CLK(ta);
            mbar_waitp(full + 8 * q, (uint32_t)((it / OZ_KS) & 1));
            OZ_CLK(tb);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t d0 = sdesc_sw64(sbase + q * kStage);  // descriptors differ only in the address field
            // A_s B_t^T for all t < NS - s in as few MMAs as possible: the B slice tiles are stacked
            // in shared memory (same 8-row-group stride), so one MMA of N = 64 m reads B_t0..B_t0+m-1
            // and writes 64 m consecutive TMEM columns starting at level s + t0's accumulator, i.e.
            // each product lands in its level (s + t). Fewer, wider MMAs read A_s once per 4 levels
            // instead of once per level (the N = 64 MMA is shared-memory-bandwidth bound).
#pragma unroll
            for (int kk = 0; kk < OZ_KC / 32; ++kk)
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int t0 = 0; t0 < NS - s; t0 += 4) {
                        const int m = (NS - s - t0) < 4 ? (NS - s - t0) : 4;
                        const uint64_t da = d0 + (uint64_t)((s * kA + kk * 32) >> 4);
                        const uint64_t db = d0 + (uint64_t)((NS * kA + t0 * kB + kk * 32) >> 4);
                        // s = 0 (t0 = 0 and 4) covers every level: it overwrites them at the first K step
                        const uint32_t accum = (kc > 0 || kk > 0 || s > 0) ? 1u : 0u;
                        mma_i8(tmem + (uint32_t)((s + t0) * OZ_N), da, db, idesc_i8(m * OZ_N), accum);
                    }
            mma_commit(empty + 8 * q);  // the stage is free once these MMAs are done
            if (FUSED && ph == 0 && kc == nk - 1) mma_commit(re_full);
            OZ_CLK(tc);
            OZ_ADD(0, ta, tb);
            OZ_ADD(1, tb, tc);
        }
        mma_commit(done);
        OZ_P(2);
    } else if (FUSED && warp >= 4) {  // park the real part: 4 column blocks, fp64 as 2 x 32 bits
        mbar_waitp(re_full, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
        for (int q = 0; q < OZ_N / 16; ++q) {
            double v[16];
            level_values16<NS>(lane_addr, q, ei, eys, v);
            uint32_t w[32];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                w[2 * c] = __double2loint(v[c]);
                w[2 * c + 1] = __double2hiint(v[c]);
            }
            tmem_st32(lane_addr + (uint32_t)(kReCol + 32 * q), w);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(re_free) : "memory");
    }
#ifdef MCINV_OZ_PROF
    if ((warp == 1 && lane == 0) || threadIdx.x == 0)
        for (int b = 0; b < 4; ++b) atomicAdd(&g_oz_prof[b], (unsigned long long)prof_[b]);
    if (threadIdx.x == 0) atomicAdd(&g_oz_prof[4], 1ull);
#endif
    __syncwarp();
    mbar_waitp(done, 0);
    OZ_P(3);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warp w reads TMEM lanes 32(w % 4).. = tile rows, columns 32(w / 4).. (16 columns of
    // all NS levels at a time). The scaled tile is staged in shared memory (the ring is free: every
    // copy was consumed and every MMA has completed) and then added into A_g: each warp takes 16
    // rows, their loads in flight at once.
    OZ_P(4);
    if constexpr (FUSED) {
        constexpr int kLd = OZ_N + 1;  // odd stride in 16-byte elements: conflict-free quarter-warps
        double2 *tile = reinterpret_cast<double2 *>(base);
#pragma unroll 1
        for (int q = ch * (OZ_N / 32); q < (ch + 1) * (OZ_N / 32); ++q) {
            double im[16];
            level_values16<NS>(lane_addr, q, ei, eys, im);
            uint32_t w[32];
            tmem_ld32(lane_addr + (uint32_t)(kReCol + 32 * q), w);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int c = 0; c < 16; ++c)
                tile[r * kLd + q * 16 + c] = make_double2(__hiloint2double(w[2 * c + 1], w[2 * c]), im[c]);
        }
        __syncthreads();
        OZ_P(5);
        const int ja = j0 + lane, jb = j0 + lane + 32;
        const bool oka = ja < n, okb = jb < n;
#pragma unroll 1
        for (int rb = warp * 16; rb < warp * 16 + 16; rb += 8) {
            double2 va[8], vb[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int ii = i0 + rb + k;
                const double2 *row = reinterpret_cast<const double2 *>(out) + (int64_t)ii * n;
                va[k] = (ii < n && oka) ? __ldcs(row + ja) : make_double2(0.0, 0.0);
                vb[k] = (ii < n && okb) ? __ldcs(row + jb) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int ii = i0 + rb + k;
                double2 *row = reinterpret_cast<double2 *>(out) + (int64_t)ii * n;
                const double2 ta = tile[(rb + k) * kLd + lane], tb = tile[(rb + k) * kLd + lane + 32];
                if (ii < n && oka) __stcs(row + ja, make_double2(va[k].x + ta.x, va[k].y + ta.y));
                if (ii < n && okb) __stcs(row + jb, make_double2(vb[k].x + tb.x, vb[k].y + tb.y));
            }
        }
    } else {
        constexpr int kLd = OZ_N + 1;  // odd stride in doubles: two lanes per bank pair at most
        double *tile = reinterpret_cast<double *>(base);
#pragma unroll 1
        for (int q = ch * (OZ_N / 32); q < (ch + 1) * (OZ_N / 32); ++q) {
            double v[16];
            level_values16<NS>(lane_addr, q, ei, eys, v);
#pragma unroll
            for (int c = 0; c < 16; ++c) tile[r * kLd + q * 16 + c] = v[c];
        }
        __syncthreads();
        OZ_P(5);
        const int ja = j0 + lane, jb = j0 + lane + 32;
        const bool oka = ja < n, okb = jb < n;
#pragma unroll 1
        for (int rb = warp * 16; rb < warp * 16 + 16; rb += 16) {
            double va[16], vb[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int ii = i0 + rb + k;
                const double *row = out + ((int64_t)ii * n) * e + part;
                va[k] = (ii < n && oka) ? __ldcs(row + (int64_t)ja * e) : 0.0;
                vb[k] = (ii < n && okb) ? __ldcs(row + (int64_t)jb * e) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int ii = i0 + rb + k;
                double *row = out + ((int64_t)ii * n) * e + part;
                if (ii < n && oka) __stcs(row + (int64_t)ja * e, va[k] + tile[(rb + k) * kLd + lane]);
                if (ii < n && okb) __stcs(row + (int64_t)jb * e, vb[k] + tile[(rb + k) * kLd + lane + 32]);
            }
        }
    }
    OZ_P(6);
#ifdef MCINV_OZ_PROF
    if (threadIdx.x == 0)
        for (int k = 1; k <= 6; ++k) atomicAdd(&g_oz_prof[4 + k], (unsigned long long)(ph_[k] - ph_[k - 1]));
#endif
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    return enc;
}

// slices [NS][n][Kp] int8 as a 3-D tensor (k', row, slice), box {64, rows, 1}, 64-B swizzle
bool slice_map(CUtensorMap *m, const int8_t *base, int n, int Kp, int ns, int rows) {
    auto enc = encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)n, (cuuint64_t)ns};
    const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)n * Kp};
    const cuuint32_t box[3] = {(cuuint32_t)OZ_KC, (cuuint32_t)rows, 1u};
    const cuuint32_t es[3] = {1u, 1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, OZ_KC == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr int kNS = 6;  // digits: 42 bits below the row scale (6 x 64 TMEM columns)

bool use_bulk() {
    if (OZ_KC != 64) return false;
    static const bool b = [] {
        const char *v = std::getenv("MCINV_OZ_BULK");
        return v == nullptr || std::atoi(v) != 0;
    }();
    return b;
}

}  // namespace

namespace {
constexpr int kBatch = 8;  // SE groups sliced per pass (tiled layout)

size_t ozaki_slot(int n, int K, bool cplx, size_t *plane_out = nullptr) {
    const size_t Kp = cplx ? 2 * (((size_t)K + OZ_KC / 2 - 1) / (OZ_KC / 2) * (OZ_KC / 2))
                           : ((size_t)K + OZ_KC - 1) / OZ_KC * OZ_KC;
    const size_t np = ((size_t)n + OZ_M - 1) / OZ_M * OZ_M;  // rows padded to the panel height
    const size_t plane = (size_t)kNS * np * Kp;
    if (plane_out) *plane_out = plane;
    return ((cplx ? 3 : 2) * plane + 2 * (size_t)n * sizeof(int) + 1023) / 1024 * 1024;
}
}  // namespace

// one slot per SE group of a slicing batch: [A | B | (A2)] digit planes, then e_i and f_j
size_t contract_ozaki_scratch(int n, int K, bool cplx, int groups) {
    const int nb = use_bulk() ? (groups < kBatch ? groups : kBatch) : 1;
    return (size_t)(nb > 0 ? nb : 1) * ozaki_slot(n, K, cplx);
}

template <typename S>
bool launch_contract_ozaki(const S *x, const S *y, double *acc, int n, int ld, int chains, int gs, int T,
                           void *scratch, size_t scratch_bytes, cudaStream_t st) {
    constexpr bool kC = ScalarTraits<S>::kDoubles == 2;
    const int K = T * gs, G = chains / gs;
    const int Kp = kC ? 2 * ((K + OZ_KC / 2 - 1) / (OZ_KC / 2) * (OZ_KC / 2)) : (K + OZ_KC - 1) / OZ_KC * OZ_KC;
    if (scratch_bytes < contract_ozaki_scratch(n, K, kC, G)) return false;
    // every level sums at most NS products of Kp digit pairs, |digit| <= 127: exact in int32
    if ((double)kNS * Kp * 127.0 * 127.0 >= 2147483648.0) return false;
    const bool bulk = use_bulk();
    size_t plane = 0;
    const size_t slot = ozaki_slot(n, K, kC, &plane);
    char *sc = static_cast<char *>(scratch);
    auto A_of = [&](int b) { return reinterpret_cast<int8_t *>(sc + b * slot); };
    auto B_of = [&](int b) { return A_of(b) + plane; };
    auto A2_of = [&](int b) { return kC ? A_of(b) + 2 * plane : nullptr; };
    auto ex_of = [&](int b) { return reinterpret_cast<int *>(sc + b * slot + (kC ? 3 : 2) * plane); };
    auto ey_of = [&](int b) { return ex_of(b) + n; };
    CUtensorMap ma{}, mb{}, ma2{};
    if (!bulk) {  // one slot, tensor maps over its planes
        if (!slice_map(&ma, A_of(0), n, Kp, kNS, OZ_M) || !slice_map(&mb, B_of(0), n, Kp, kNS, OZ_N)) return false;
        if (kC && !slice_map(&ma2, A2_of(0), n, Kp, kNS, OZ_M)) return false;
    }
    const size_t smem = (size_t)OZ_KS * kNS * (OZ_M + OZ_N) * OZ_KC + 16 * OZ_KS + 32 + OZ_N * sizeof(int) + 1024;
    const bool fused = kC && bulk;  // complex: real and imaginary parts in one CTA
    auto kg = fused ? ozaki_gemm_kernel<kNS, true, true>
                    : (bulk ? ozaki_gemm_kernel<kNS, true, false> : ozaki_gemm_kernel<kNS, false, false>);
    if (cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
    const dim3 grid((n + OZ_N - 1) / OZ_N, (n + OZ_M - 1) / OZ_M);
    const int e = kC ? 2 : 1;
    // tiled: X panels of 128 rows, Y panels of 64 (both padded within the np-row plane)
    const int rx = bulk ? (n + OZ_M - 1) / OZ_M * OZ_M : n, ry = bulk ? (n + OZ_N - 1) / OZ_N * OZ_N : n;
    const int batch = bulk ? kBatch : 1;
    for (int g0 = 0; g0 < G; g0 += batch) {
        const int nb = G - g0 < batch ? G - g0 : batch;
        if (bulk) {
            ozaki_slice_tiled_kernel<S, kNS><<<dim3(nb, rx), 128, 0, st>>>(x, n, ld, gs, g0, K, Kp, A_of(0), A2_of(0),
                                                                       ex_of(0), OZ_M, slot);
            ozaki_slice_tiled_kernel<S, kNS><<<dim3(nb, ry), 128, 0, st>>>(y, n, ld, gs, g0, K, Kp, B_of(0), nullptr,
                                                                       ey_of(0), OZ_N, slot);
        } else {
            ozaki_slice_kernel<S, kNS><<<rx, 256, 0, st>>>(x, n, ld, gs, g0, K, Kp, A_of(0), A2_of(0), ex_of(0), 0, OZ_M);
            ozaki_slice_kernel<S, kNS><<<ry, 256, 0, st>>>(y, n, ld, gs, g0, K, Kp, B_of(0), nullptr, ey_of(0), 0, OZ_N);
        }
        for (int b = 0; b < nb; ++b) {
            double *out = acc + (int64_t)(g0 + b) * n * n * e;
            if (fused) {
                kg<<<grid, 256, smem, st>>>(ma, mb, A_of(b), A2_of(b), B_of(b), ex_of(b), ey_of(b), out, n, e, 0, Kp);
            } else {
                kg<<<grid, 256, smem, st>>>(ma, mb, A_of(b), nullptr, B_of(b), ex_of(b), ey_of(b), out, n, e, 0, Kp);
                if (kC)
                    kg<<<grid, 256, smem, st>>>(ma2, mb, A2_of(b), nullptr, B_of(b), ex_of(b), ey_of(b), out, n, e, 1,
                                                Kp);
            }
        }
    }
#ifdef MCINV_OZ_PROF
    {
        unsigned long long h[12];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_oz_prof, sizeof h);
        const double c = h[4] ? (double)h[4] * (Kp / OZ_KC) : 1.0;
        fprintf(stderr, "ozaki prof: per chunk cycles: MMA thread wait-full %.0f mma-issue %.0f; producer wait-empty %.0f copy-issue %.0f (CTAs %llu)\n",
                h[0] / c, h[1] / c, h[2] / c, h[3] / c, h[4]);
        const double cc = h[4] ? (double)h[4] : 1.0;
        fprintf(stderr, "ozaki prof: per CTA cycles: prologue %.0f mainloop %.0f drain %.0f tmem-ld %.0f stage %.0f rmw %.0f\n",
                h[5] / cc, h[6] / cc, h[7] / cc, h[8] / cc, h[9] / cc, h[10] / cc);
        const unsigned long long z[12] = {};
        cudaMemcpyToSymbol(g_oz_prof, z, sizeof z);
    }
#endif
    // launched: a launch error stays pending for the caller's check (no fallback may add the
    // same samples a second time)
    return true;
}

template bool launch_contract_ozaki<double>(const double *, const double *, double *, int, int, int, int, int, void *,
                                            size_t, cudaStream_t);
template bool launch_contract_ozaki<cd>(const cd *, const cd *, double *, int, int, int, int, int, void *, size_t,
                                        cudaStream_t);

}  // namespace mcinv
