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
// GEMM tile 128 x 64 (UMMA M = 128, N = 64, K = 32), K staged in chunks of 64 int8 per slice by
// TMA (64-B swizzle, K-major), all NS slices of both operands per stage, a ring of KS stages.
// One thread issues the TMA copies and the MMAs; tcgen05.commit frees a stage; four warps read the
// NS accumulators (tcgen05.ld) in the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

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
template <typename S, int NS>
__global__ void ozaki_slice_kernel(const S *__restrict__ snap, int n, int ld, int gs, int g, int K, int Kp,
                                   int8_t *__restrict__ out, int8_t *__restrict__ out2, int *__restrict__ expo) {
    constexpr bool CPLX = ScalarTraits<S>::kDoubles == 2;
    const int i = blockIdx.x;
    __shared__ double red[32];
    double mx = 0.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
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
    if (threadIdx.x == 0) expo[i] = e;
    const size_t plane = (size_t)n * Kp;
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
        if (k < K) {
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
                    out[s * plane + (size_t)i * Kp + k] = d0[s];
                    out[s * plane + (size_t)i * Kp + Kh + k] = d1[s];
                    if (out2) {
                        out2[s * plane + (size_t)i * Kp + k] = d1[s];
                        out2[s * plane + (size_t)i * Kp + Kh + k] = static_cast<int8_t>(-d0[s]);
                    }
                }
            }
        } else {
#pragma unroll
            for (int s = 0; s < NS; ++s) out[s * plane + (size_t)i * Kp + k] = d0[s];
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
// instruction descriptor: s8 x s8 -> s32, K-major A and B, N = 64, M = 128
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_N >> 3) << 17) |
                              ((uint32_t)(OZ_M >> 4) << 24);
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    const uint32_t mask0 = 0, mask1 = 0, mask2 = 0, mask3 = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdescI8), "r"(acc), "r"(mask0), "r"(mask1), "r"(mask2), "r"(mask3));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// ---------------------------------------------------------------- GEMM + epilogue
// out: A_g (fp64, e doubles per element, stride e): out[(i n + j) e + part] += sum_L 2^(ei + fj - 7(L+2)) D_L[i][j]
template <int NS>
__global__ void __launch_bounds__(128, 1) ozaki_gemm_kernel(const __grid_constant__ CUtensorMap ma,
                                                            const __grid_constant__ CUtensorMap mb,
                                                            const int *__restrict__ ex, const int *__restrict__ ey,
                                                            double *__restrict__ out, int n, int e, int part, int Kp) {
    constexpr uint32_t kA = OZ_M * OZ_KC, kB = OZ_N * OZ_KC;  // bytes of one slice tile
    constexpr uint32_t kStage = NS * (kA + kB);
    extern __shared__ __align__(128) unsigned char smo[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smo) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = s_addr(base);
    const uint32_t full = sbase + OZ_KS * kStage, empty = full + 8 * OZ_KS, done = empty + 8 * OZ_KS;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(base + OZ_KS * kStage + 16 * OZ_KS + 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.y * OZ_M, j0 = blockIdx.x * OZ_N;
    const int nk = Kp / OZ_KC;
    if (threadIdx.x == 0) {
        for (int q = 0; q < OZ_KS; ++q) {
            mbar_init1(full + 8 * q);
            mbar_init1(empty + 8 * q);
        }
        mbar_init1(done);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // 512 TMEM columns: NS accumulators of N = 64 int32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(tmem_slot);

    if (threadIdx.x == 0) {
        auto issue = [&](int kc) {
            const int q = kc % OZ_KS;
            const uint32_t st = sbase + q * kStage;
            mbar_expect(full + 8 * q, kStage);
            for (int s = 0; s < NS; ++s) {
                tma3(st + s * kA, &ma, kc * OZ_KC, i0, s, full + 8 * q);
                tma3(st + NS * kA + s * kB, &mb, kc * OZ_KC, j0, s, full + 8 * q);
            }
        };
        for (int kc = 0; kc < OZ_KS && kc < nk; ++kc) issue(kc);
        for (int kc = 0; kc < nk; ++kc) {
            const int q = kc % OZ_KS;
            mbar_waitp(full + 8 * q, (uint32_t)((kc / OZ_KS) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t d0 = sdesc_sw64(sbase + q * kStage);  // descriptors differ only in the address field
#pragma unroll
            for (int t = 0; t < NS; ++t)
#pragma unroll
                for (int s = 0; s + t < NS; ++s) {
                    const uint32_t acc_col = tmem + (uint32_t)((s + t) * OZ_N);
#pragma unroll
                    for (int kk = 0; kk < OZ_KC / 32; ++kk) {
                        const uint64_t da = d0 + (uint64_t)((s * kA + kk * 32) >> 4);
                        const uint64_t db = d0 + (uint64_t)((NS * kA + t * kB + kk * 32) >> 4);
                        // the first product of each level (t = 0 of the first chunk) overwrites it
                        const uint32_t accum = (kc > 0 || kk > 0 || t > 0) ? 1u : 0u;
                        mma_i8(acc_col, da, db, accum);
                    }
                }
            mma_commit(empty + 8 * q);  // the stage is free once these MMAs are done
            // refill the PREVIOUS chunk's stage: its MMAs are done by now (the tensor pipe is busy
            // with this chunk's), so waiting on it does not drain the MMA queue
            if (kc >= 1 && kc - 1 + OZ_KS < nk) {
                const int pq = (kc - 1) % OZ_KS;
                mbar_waitp(empty + 8 * pq, (uint32_t)(((kc - 1) / OZ_KS) & 1));
                issue(kc - 1 + OZ_KS);
            }
        }
        mma_commit(done);
    }
    __syncwarp();
    mbar_waitp(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warp w reads TMEM lanes 32w..32w+31 = tile rows; 64 columns per level
    const int r = warp * 32 + lane, i = i0 + r;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    double sum[OZ_N];
#pragma unroll
    for (int c = 0; c < OZ_N; ++c) sum[c] = 0.0;
    for (int L = NS - 1; L >= 0; --L) {  // smallest terms first
        uint32_t v[OZ_N];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
            "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"
            "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
              "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]), "=r"(v[38]), "=r"(v[39]),
              "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]), "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]),
              "=r"(v[48]), "=r"(v[49]), "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
              "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]), "=r"(v[62]), "=r"(v[63])
            : "r"(lane_addr + (uint32_t)(L * OZ_N)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const double w = ldexp(1.0, -7 * (L + 2));
#pragma unroll
        for (int c = 0; c < OZ_N; ++c) sum[c] = fma(static_cast<double>(static_cast<int32_t>(v[c])), w, sum[c]);
    }
    if (i < n) {
        const int ei = ex[i];
        double *row = out + ((int64_t)i * n) * e + part;
#pragma unroll
        for (int c = 0; c < OZ_N; ++c) {
            const int j = j0 + c;
            if (j < n) row[(int64_t)j * e] += ldexp(sum[c], ei + ey[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
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

}  // namespace

size_t contract_ozaki_scratch(int n, int K, bool cplx) {
    const size_t Kp = cplx ? 2 * (((size_t)K + OZ_KC / 2 - 1) / (OZ_KC / 2) * (OZ_KC / 2))
                           : ((size_t)K + OZ_KC - 1) / OZ_KC * OZ_KC;
    const size_t plane = (size_t)kNS * n * Kp;
    return (cplx ? 3 : 2) * plane + 2 * (size_t)n * sizeof(int) + 1024;
}

template <typename S>
bool launch_contract_ozaki(const S *x, const S *y, double *acc, int n, int ld, int chains, int gs, int T,
                           void *scratch, size_t scratch_bytes, cudaStream_t st) {
    constexpr bool kC = ScalarTraits<S>::kDoubles == 2;
    const int K = T * gs;
    const int Kp = kC ? 2 * ((K + OZ_KC / 2 - 1) / (OZ_KC / 2) * (OZ_KC / 2)) : (K + OZ_KC - 1) / OZ_KC * OZ_KC;
    if (scratch_bytes < contract_ozaki_scratch(n, K, kC)) return false;
    const size_t plane = (size_t)kNS * n * Kp;
    int8_t *A = static_cast<int8_t *>(scratch), *B = A + plane, *A2 = kC ? B + plane : nullptr;
    int *ex = reinterpret_cast<int *>(reinterpret_cast<char *>(scratch) + (kC ? 3 : 2) * plane);
    int *ey = ex + n;
    CUtensorMap ma, mb, ma2;
    if (!slice_map(&ma, A, n, Kp, kNS, OZ_M) || !slice_map(&mb, B, n, Kp, kNS, OZ_N)) return false;
    if (kC && !slice_map(&ma2, A2, n, Kp, kNS, OZ_M)) return false;
    const size_t smem = (size_t)OZ_KS * kNS * (OZ_M + OZ_N) * OZ_KC + 16 * OZ_KS + 16 + 1024;
    auto kg = ozaki_gemm_kernel<kNS>;
    if (cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
    const dim3 grid((n + OZ_N - 1) / OZ_N, (n + OZ_M - 1) / OZ_M);
    const int e = kC ? 2 : 1;
    for (int g = 0; g < chains / gs; ++g) {
        double *out = acc + (int64_t)g * n * n * e;
        ozaki_slice_kernel<S, kNS><<<n, 256, 0, st>>>(x, n, ld, gs, g, K, Kp, A, A2, ex);
        ozaki_slice_kernel<S, kNS><<<n, 256, 0, st>>>(y, n, ld, gs, g, K, Kp, B, nullptr, ey);
        kg<<<grid, 128, smem, st>>>(ma, mb, ex, ey, out, n, e, 0, Kp);
        if (kC) kg<<<grid, 128, smem, st>>>(ma2, mb, ex, ey, out, n, e, 1, Kp);
    }
    return cudaGetLastError() == cudaSuccess;
}

template bool launch_contract_ozaki<double>(const double *, const double *, double *, int, int, int, int, int, void *,
                                            size_t, cudaStream_t);
template bool launch_contract_ozaki<cd>(const cd *, const cd *, double *, int, int, int, int, int, void *, size_t,
                                        cudaStream_t);

}  // namespace mcinv
