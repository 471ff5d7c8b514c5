// contract.cu -- K3: the full-inverse accumulation X Y^dagger on FP64 tensor
// cores (DMMA, mma.sync.m8n8k4.f64; tcgen05 has no f64 kind).
//
// After each chunk of T sampling sweeps the sweep kernel has stored the
// states Z, W of every chain in X[t][i][c], Y[t][j][c]. For each standard-
// error group g (gs consecutive chains) this kernel adds
//     A_g[i][j] += sum_{t < T} sum_{c in g} X[t][i][c] * conj(Y[t][j][c])
// i.e. sum_k z^(k) w^(k)dagger of Eq. (1/C), as a GEMM with
// K = T * gs. Complex: Re A += Xr Yr^T + Xi Yi^T, Im A += Xi Yr^T - Xr Yi^T
// (four real DMMA products per complex 8x8x4 step).
//
// CTA tile 64 x 64 outputs (4 warps, 32 x 32 each), K staged in chunks of
// KC = 16 by cp.async into a double-buffered shared-memory pipeline, k-major
// with a padded row stride so the m8n8k4 fragment loads (lane -> row = lane/4,
// k = lane%4) are bank-conflict free; complex values stay interleaved (one
// 16-B shared load gives both parts of a fragment element).
#include <cuda.h>  // CUtensorMap (types only: the encoder comes from cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>

#include <cstdlib>

#include "mcinv_internal.cuh"
#include "scalar.cuh"

namespace mcinv {

namespace {

constexpr int BM = 64, BN = 64, KC = 16;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async(void *smem, const void *gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int bytes = pred ? 16 : 0;  // src-size 0: zero-fill (rows past n, k past K)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int bytes = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// shared tile: [KC][row stride] elements; stride chosen conflict-free for the fragment pattern
template <typename S> struct Tile;
template <> struct Tile<double> { static constexpr int LD = BM + 4; };  // 8-B elements
template <> struct Tile<cd> { static constexpr int LD = BM + 2; };      // 16-B elements

template <typename S, int NTH>
__device__ __forceinline__ void stage(S *sm, const S *g, int t0k, int i0, int n, int ld, int gs, int c0, int K,
                                     int tid) {
    // element (k, r) of the chunk = g[((t) * n + i0 + r) * ld + c0 + c], k = t0k + kk, t = k / gs, c = k % gs
    constexpr int LDS = Tile<S>::LD;
    static_assert(NTH % KC == 0, "a thread keeps its k column");
    const int kk = tid % KC, r0 = tid / KC;
    constexpr int RSTEP = NTH / KC;
    const int k = t0k + kk;
    if (gs % KC == 0) {
        // the chunk lies in one snapshot sweep t (KC divides gs): one division per chunk,
        // then a row stride per element (the staging was integer-bound with a division each)
        const int t = t0k / gs, c = t0k - t * gs + kk;
        const S *src = g + ((int64_t)t * n + i0 + r0) * ld + c0 + c;
        const int64_t step = (int64_t)RSTEP * ld;
#pragma unroll 4
        for (int r = r0; r < BM; r += RSTEP, src += step) {
            const bool ok = i0 + r < n;
            const S *q = ok ? src : g;
            if constexpr (ScalarTraits<S>::kDoubles == 2) cp_async(sm + kk * LDS + r, q, ok);
            else cp_async8(sm + kk * LDS + r, q, ok);
        }
        return;
    }
    const bool okk = k < K;
    const int t = okk ? k / gs : 0, c = okk ? k % gs : 0;
    for (int r = r0; r < BM; r += RSTEP) {
        const bool ok = okk && i0 + r < n;
        const S *src = g + ((int64_t)t * n + (ok ? i0 + r : 0)) * ld + c0 + c;
        if constexpr (ScalarTraits<S>::kDoubles == 2) cp_async(sm + kk * LDS + r, src, ok);
        else cp_async8(sm + kk * LDS + r, src, ok);
    }
}

// WN: output columns per warp (32: 4 warps of 32 x 32; 16: 8 warps of 32 x 16, half the
// accumulator registers per thread and twice the warps per SM)
// M3 (complex only): the 3-multiplication form of x conj(y) -- P1 = xr yr, P2 = xi yi,
// P3 = (xr + xi)(yr - yi); Re = P1 + P2, Im = P3 - P1 + P2 -- three real DMMA products per
// complex one instead of four (the DMMA pipe is the bound)
template <typename S, bool CPLX, int WN, bool M3>
__global__ void __launch_bounds__(32 * 2 * (BN / WN)) contract_kernel(const S *__restrict__ x, const S *__restrict__ y,
                                                                    double *__restrict__ acc, int n, int ld, int gs,
                                                                    int T) {
    constexpr int LDS = Tile<S>::LD;
    constexpr int NTH = 32 * 2 * (BN / WN);
    constexpr int NB = WN / 8;  // 8-column tiles per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S *xs = reinterpret_cast<S *>(smem_raw);  // [2][KC][LDS]
    S *ys = xs + 2 * KC * LDS;                // [2][KC][LDS]
    const int g = blockIdx.z;
    const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * WN;
    const int K = T * gs, c0 = g * gs;
    double cr[4][NB][2], ci[4][NB][2];
    constexpr int A3 = M3 ? 4 : 1, B3 = M3 ? NB : 1;
    double c3[A3][B3][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
#pragma unroll
    for (int a = 0; a < A3; ++a)
#pragma unroll
        for (int b = 0; b < B3; ++b) c3[a][b][0] = c3[a][b][1] = 0.0;

    const int nk = (K + KC - 1) / KC;
    stage<S, NTH>(xs, x, 0, i0, n, ld, gs, c0, K, tid);
    stage<S, NTH>(ys, y, 0, j0, n, ld, gs, c0, K, tid);
    cp_commit();
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nk) {
            stage<S, NTH>(xs + (buf ^ 1) * KC * LDS, x, (kc + 1) * KC, i0, n, ld, gs, c0, K, tid);
            stage<S, NTH>(ys + (buf ^ 1) * KC * LDS, y, (kc + 1) * KC, j0, n, ld, gs, c0, K, tid);
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const S *xb = xs + buf * KC * LDS, *yb = ys + buf * KC * LDS;
#pragma unroll
        for (int ks = 0; ks < KC; ks += 4) {
            const int kk = ks + (lane & 3);
            S av[4], bv[NB];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = xb[kk * LDS + wm + a * 8 + (lane >> 2)];
#pragma unroll
            for (int b = 0; b < NB; ++b) bv[b] = yb[kk * LDS + wn + b * 8 + (lane >> 2)];
            // four passes over the 4 x NB tiles: consecutive DMMAs never share an accumulator
            if constexpr (CPLX && M3) {
                double sa[4], db[NB];
#pragma unroll
                for (int a = 0; a < 4; ++a) sa[a] = av[a].re + av[a].im;
#pragma unroll
                for (int b = 0; b < NB; ++b) db[b] = bv[b].re - bv[b].im;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a].re, bv[b].re);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(ci[a][b][0], ci[a][b][1], av[a].im, bv[b].im);
#pragma unroll
                for (int a = 0; a < A3; ++a)
#pragma unroll
                    for (int b = 0; b < B3; ++b) dmma(c3[a][b][0], c3[a][b][1], sa[a], db[b]);
            } else if constexpr (CPLX) {
                double na[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) na[a] = -av[a].re;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a].re, bv[b].re);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(ci[a][b][0], ci[a][b][1], av[a].im, bv[b].re);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a].im, bv[b].im);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(ci[a][b][0], ci[a][b][1], na[a], bv[b].im);
            } else {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a], bv[b]);
            }
        }
        __syncthreads();
    }
    if constexpr (M3) {  // Re = P1 + P2, Im = P3 - P1 + P2
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double p1 = cr[a][b][h], p2 = ci[a][b][h];
                    cr[a][b][h] = p1 + p2;
                    ci[a][b][h] = c3[a < A3 ? a : 0][b < B3 ? b : 0][h] - p1 + p2;
                }
    }
    // accumulate into A_g (layout [G][n][n] x e doubles): each lane owns 2 adjacent columns
    const int e = CPLX ? 2 : 1;
    double *out = acc + (int64_t)g * n * n * e;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int i = i0 + wm + a * 8 + (lane >> 2);
            const int j = j0 + wn + b * 8 + (lane & 3) * 2;
            if (i >= n) continue;
            double *p = out + ((int64_t)i * n + j) * e;
            if (CPLX) {
                if (j + 1 < n) {
                    double4 v = *reinterpret_cast<double4 *>(p);
                    v.x += cr[a][b][0];
                    v.y += ci[a][b][0];
                    v.z += cr[a][b][1];
                    v.w += ci[a][b][1];
                    *reinterpret_cast<double4 *>(p) = v;
                } else if (j < n) {
                    p[0] += cr[a][b][0];
                    p[1] += ci[a][b][0];
                }
            } else {
                if (j + 1 < n && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
                    double2 v = *reinterpret_cast<double2 *>(p);
                    v.x += cr[a][b][0];
                    v.y += cr[a][b][1];
                    *reinterpret_cast<double2 *>(p) = v;
                } else {
                    if (j < n) p[0] += cr[a][b][0];
                    if (j + 1 < n) p[1] += cr[a][b][1];
                }
            }
        }
}

// ---------------------------------------------------------------- TMA-staged variant
//
// The same contraction with its operand tiles moved by the tensor-memory accelerator:
// X (and Y) is the 3-D tensor (chain, row, snapshot sweep) of 8- or 16-B elements; a
// k-chunk of KC = 16 lies in one snapshot sweep (group size a multiple of 16), so a stage
// is, per operand, the box {16 chains, 64 rows, 1 sweep} -- two boxes of 8 chains for
// complex (a 128-B swizzle span holds 8) -- landing in shared memory with the 128-B
// swizzle (16-B chunk c of row r at chunk c ^ (r & 7): the m8n8k4 fragment reads, 8 rows x
// 4 k, hit 32 distinct banks). A ring of KS stages; thread 0 issues the bulk tensor copies
// (cp.async.bulk.tensor, SASS UTMALDG) onto the stage's mbarrier; rows past n arrive as
// zeros (out-of-bounds fill).
constexpr int KS = 3;  // stages in flight

template <typename S> struct TmaTile;
template <> struct TmaTile<double> { static constexpr int kBoxes = 1, kBoxElems = 16; };
template <> struct TmaTile<cd> { static constexpr int kBoxes = 2, kBoxElems = 8; };

__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
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

template <typename S, bool CPLX, int WN, bool M3>
__global__ void __launch_bounds__(32 * 2 * (BN / WN), 2) contract_tma_kernel(const __grid_constant__ CUtensorMap mx,
                                                                        const __grid_constant__ CUtensorMap my,
                                                                        double *__restrict__ acc, int n, int gs,
                                                                        int T) {
    constexpr int NB = WN / 8;
    constexpr int BOX = TmaTile<S>::kBoxElems, NBOX = TmaTile<S>::kBoxes;
    constexpr uint32_t kBoxBytes = 64 * 128;                    // 64 rows x 128 B
    constexpr uint32_t kStageBytes = 2 * NBOX * kBoxBytes;      // X and Y
    extern __shared__ __align__(128) unsigned char smem_tma[];
    // 1024-B aligned base for the swizzled boxes (1 KB of slack is allocated); the mbarriers
    // and the stage counters after the stages
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_tma) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(base));
    const uint32_t bars = sbase + KS * kStageBytes;
    // per stage: how many warps are done with it; the last one refills it (no CTA barrier)
    unsigned *done_cnt = reinterpret_cast<unsigned *>(base + KS * kStageBytes + 8 * KS);
    const int g = blockIdx.z;
    const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * WN;
    const int K = T * gs;
    const int nk = K / KC;  // gs % KC == 0
    if (tid == 0) {
        for (int q = 0; q < KS; ++q) {
            mbar_init1(bars + 8 * q);
            done_cnt[q] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&my)) : "memory");
    }
    __syncthreads();
    auto issue = [&](int kc) {  // one thread: the stage of chunk kc
        const int q = kc % KS;
        const uint32_t st = sbase + q * kStageBytes, bar = bars + 8 * q;
        const int k0 = kc * KC, t = k0 / gs, c = g * gs + (k0 - t * gs);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of this slot precede
        mbar_expect(bar, kStageBytes);
#pragma unroll
        for (int b = 0; b < NBOX; ++b) {
            // the map's innermost dimension counts doubles (two per complex chain element)
            const int cc = (c + b * BOX) * (CPLX ? 2 : 1);
            tma_load3(st + b * kBoxBytes, &mx, cc, i0, t, bar);
            tma_load3(st + (NBOX + b) * kBoxBytes, &my, cc, j0, t, bar);
        }
    };
    if (tid == 0)
        for (int kc = 0; kc < KS && kc < nk; ++kc) issue(kc);

    double cr[4][NB][2], ci[4][NB][2];
    constexpr int A3 = M3 ? 4 : 1, B3 = M3 ? NB : 1;
    double c3[A3][B3][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;
#pragma unroll
    for (int a = 0; a < A3; ++a)
#pragma unroll
        for (int b = 0; b < B3; ++b) c3[a][b][0] = c3[a][b][1] = 0.0;

    // element (row r, k) of an operand in a stage: box k / BOX, swizzled 16-B chunk
    const int rsw = lane >> 2;  // r & 7 for every fragment row (wm, wn, a * 8, b * 8 are multiples of 8)
    auto elem = [&](const unsigned char *op, int r, int kk) -> S {
        const unsigned char *bx = op + (kk / BOX) * kBoxBytes + r * 128;
        if constexpr (CPLX) {
            const double2 v = *reinterpret_cast<const double2 *>(bx + (((kk % BOX) ^ rsw) << 4));
            return S{v.x, v.y};
        } else {
            const int kb = kk % BOX;
            return *reinterpret_cast<const double *>(bx + ((((kb >> 1) ^ rsw) << 4) | ((kb & 1) << 3)));
        }
    };
    constexpr int NWARPS = 2 * (BN / WN);
    for (int kc = 0; kc < nk; ++kc) {
        const int q = kc % KS;
        mbar_wait_parity(bars + 8 * q, static_cast<uint32_t>((kc / KS) & 1));
        const unsigned char *xb = base + q * kStageBytes, *yb = xb + NBOX * kBoxBytes;
#pragma unroll
        for (int ks = 0; ks < KC; ks += 4) {
            const int kk = ks + (lane & 3);
            S av[4], bv[NB];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = elem(xb, wm + a * 8 + rsw, kk);
#pragma unroll
            for (int b = 0; b < NB; ++b) bv[b] = elem(yb, wn + b * 8 + rsw, kk);
            if constexpr (CPLX && M3) {
                double sa[4], db[NB];
#pragma unroll
                for (int a = 0; a < 4; ++a) sa[a] = av[a].re + av[a].im;
#pragma unroll
                for (int b = 0; b < NB; ++b) db[b] = bv[b].re - bv[b].im;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a].re, bv[b].re);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(ci[a][b][0], ci[a][b][1], av[a].im, bv[b].im);
#pragma unroll
                for (int a = 0; a < A3; ++a)
#pragma unroll
                    for (int b = 0; b < B3; ++b) dmma(c3[a][b][0], c3[a][b][1], sa[a], db[b]);
            } else if constexpr (CPLX) {
                double na[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) na[a] = -av[a].re;
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a].re, bv[b].re);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(ci[a][b][0], ci[a][b][1], av[a].im, bv[b].re);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a].im, bv[b].im);
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(ci[a][b][0], ci[a][b][1], na[a], bv[b].im);
            } else {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < NB; ++b) dmma(cr[a][b][0], cr[a][b][1], av[a], bv[b]);
            }
        }
        // this warp is done with stage q; the last warp to finish it refills it with chunk
        // kc + KS (its reads are ordered before the count by the fence, and the copy's async
        // writes after every counted read by the proxy fence in issue)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(done_cnt + q, 1u) == NWARPS - 1) {
                done_cnt[q] = 0;
                if (kc + KS < nk) issue(kc + KS);
            }
        }
    }
    if constexpr (M3) {  // Re = P1 + P2, Im = P3 - P1 + P2
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double p1 = cr[a][b][h], p2 = ci[a][b][h];
                    cr[a][b][h] = p1 + p2;
                    ci[a][b][h] = c3[a < A3 ? a : 0][b < B3 ? b : 0][h] - p1 + p2;
                }
    }
    const int e = CPLX ? 2 : 1;
    double *out = acc + (int64_t)g * n * n * e;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int i = i0 + wm + a * 8 + (lane >> 2);
            const int j = j0 + wn + b * 8 + (lane & 3) * 2;
            if (i >= n) continue;
            double *p = out + ((int64_t)i * n + j) * e;
            if (CPLX) {
                if (j + 1 < n) {
                    double4 v = *reinterpret_cast<double4 *>(p);
                    v.x += cr[a][b][0];
                    v.y += ci[a][b][0];
                    v.z += cr[a][b][1];
                    v.w += ci[a][b][1];
                    *reinterpret_cast<double4 *>(p) = v;
                } else if (j < n) {
                    p[0] += cr[a][b][0];
                    p[1] += ci[a][b][0];
                }
            } else {
                if (j + 1 < n && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
                    double2 v = *reinterpret_cast<double2 *>(p);
                    v.x += cr[a][b][0];
                    v.y += cr[a][b][1];
                    *reinterpret_cast<double2 *>(p) = v;
                } else {
                    if (j < n) p[0] += cr[a][b][0];
                    if (j + 1 < n) p[1] += cr[a][b][1];
                }
            }
        }
}

// The 3-D tensor map (chain, row, snapshot sweep) of one snapshot buffer; false if the
// driver entry point is unavailable or the encoding fails (the cp.async kernel then runs)
template <typename S>
bool encode_snap_map(CUtensorMap *m, const S *base, int n, int ld, int T) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!enc) return false;
    constexpr bool kC = ScalarTraits<S>::kDoubles == 2;
    const cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)n, (cuuint64_t)T};
    const cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(S), (cuuint64_t)n * ld * sizeof(S)};
    const cuuint32_t box[3] = {(cuuint32_t)TmaTile<S>::kBoxElems, 64u, 1u};
    const cuuint32_t es[3] = {1u, 1u, 1u};
    // complex elements as pairs of doubles would need a 4-D map; a 16-B element is moved as
    // CU_TENSOR_MAP_DATA_TYPE_FLOAT64 with the chain dimension doubled
    cuuint64_t d2[3] = {dims[0] * (kC ? 2 : 1), dims[1], dims[2]};
    cuuint32_t b2[3] = {box[0] * (kC ? 2u : 1u), box[1], box[2]};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<S *>(base), d2, strides, b2, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

template <typename S>
void launch_contract(const S *x, const S *y, double *acc, int n, int ld, int chains, int gs, int T,
                     cudaStream_t st) {
    const int G = chains / gs;
    dim3 grid((n + BN - 1) / BN, (n + BM - 1) / BM, G);
    const size_t smem = 2 * 2 * KC * Tile<S>::LD * sizeof(S);
    constexpr bool kC = ScalarTraits<S>::kDoubles == 2;
    // MCINV_CONTRACT_WN: output columns per warp (32: 4 warps per CTA, 16: 8 warps)
    const char *e = std::getenv("MCINV_CONTRACT_WN");
    const char *m3 = std::getenv("MCINV_CONTRACT_3M");
    // the TMA-staged kernel when a k-chunk lies in one snapshot sweep (MCINV_CONTRACT_TMA=0: cp.async)
    const char *tm = std::getenv("MCINV_CONTRACT_TMA");
    if (gs % KC == 0 && !(tm && std::atoi(tm) == 0) && !(e && std::atoi(e) == 32)) {
        CUtensorMap mx, my;
        if (encode_snap_map<S>(&mx, x, n, ld, T) && encode_snap_map<S>(&my, y, n, ld, T)) {
            const size_t smem_t = (size_t)KS * 2 * TmaTile<S>::kBoxes * 64 * 128 + 12 * KS + 1024;
            const bool use3 = kC && !(m3 && std::atoi(m3) == 0);
            auto k = use3 ? contract_tma_kernel<S, kC, 16, kC> : contract_tma_kernel<S, kC, 16, false>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
            k<<<grid, 256, smem_t, st>>>(mx, my, acc, n, gs, T);
            return;
        }
    }
    // complex: the 3-multiplication form by default (config 3: 34.2 -> 39.5 algorithmic FP64
    // TFLOP/s, i.e. 8 n^2 flops per chain-sweep counted; MCINV_CONTRACT_3M=0 for 4 products)
    if (kC && !(m3 && std::atoi(m3) == 0)) {  // 3 products per complex MAC, 8 warps of 32 x 16
        auto k = contract_kernel<S, kC, 16, kC>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 256, smem, st>>>(x, y, acc, n, ld, gs, T);
    } else if (e && std::atoi(e) == 16) {
        auto k = contract_kernel<S, kC, 16, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 256, smem, st>>>(x, y, acc, n, ld, gs, T);
    } else {
        auto k = contract_kernel<S, kC, 32, false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 128, smem, st>>>(x, y, acc, n, ld, gs, T);
    }
}

template void launch_contract<double>(const double *, const double *, double *, int, int, int, int, int,
                                      cudaStream_t);
template void launch_contract<cd>(const cd *, const cd *, double *, int, int, int, int, int, cudaStream_t);

}  // namespace mcinv
