// contract.cu -- K3: the full-inverse accumulation X Y^dagger on FP64 tensor
// cores (DMMA, mma.sync.m8n8k4.f64; tcgen05 has no f64 kind).
//
// After each chunk of T sampling sweeps the sweep kernel has stored the
// states Z, W of every chain in X[t][i][c], Y[t][j][c]. For each standard-
// error group g (gs consecutive chains) this kernel adds
//     A_g[i][j] += sum_{t < T} sum_{c in g} X[t][i][c] * conj(Y[t][j][c])
// i.e. sum_k z^(k) w^(k)dagger of Eq. (1/C), as a GEMM with
// K = T * gs. Complex: Re A += Xr Yr^T + Xi Yi^T, Im A += Xi Yr^T - Xr Yi^T.
#include "mcinv_internal.cuh"
#include "scalar.cuh"

namespace mcinv {

namespace {

constexpr int BM = 64, BN = 64, KC = 16, PADK = KC + 1;

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double re_of(double v) { return v; }
__device__ __forceinline__ double im_of(double) { return 0.0; }
__device__ __forceinline__ double re_of(cd v) { return v.re; }
__device__ __forceinline__ double im_of(cd v) { return v.im; }

template <typename S, bool CPLX>
__global__ void __launch_bounds__(128) contract_kernel(const S *__restrict__ x, const S *__restrict__ y,
                                                      double *__restrict__ acc, int n, int ld, int gs, int T) {
    __shared__ double xr[BM][PADK], yr[BN][PADK];
    __shared__ double xi[CPLX ? BM : 1][PADK], yi[CPLX ? BN : 1][PADK];
    const int g = blockIdx.z;
    const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int K = T * gs;
    double cr[4][4][2], ci[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) cr[a][b][0] = cr[a][b][1] = ci[a][b][0] = ci[a][b][1] = 0.0;

    for (int k0 = 0; k0 < K; k0 += KC) {
        // stage X[i0:i0+64, k0:k0+KC] and Y[j0:j0+64, k0:k0+KC]
        for (int e = threadIdx.x; e < BM * KC; e += blockDim.x) {
            const int r = e / KC, kk = e % KC, k = k0 + kk;
            const int t = k / gs, c = g * gs + k % gs;
            S vx = zero_s<S>(), vy = zero_s<S>();
            if (k < K) {
                if (i0 + r < n) vx = x[((int64_t)t * n + i0 + r) * ld + c];
                if (j0 + r < n) vy = y[((int64_t)t * n + j0 + r) * ld + c];
            }
            xr[r][kk] = re_of(vx);
            yr[r][kk] = re_of(vy);
            if constexpr (CPLX) {
                xi[r][kk] = im_of(vx);
                yi[r][kk] = im_of(vy);
            }
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < KC; ks += 4) {
            const int ka = ks + (lane & 3);
            double ar[4], br[4], ai[4], bi[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                ar[a] = xr[wm + a * 8 + (lane >> 2)][ka];
                br[a] = yr[wn + a * 8 + (lane >> 2)][ka];
                if constexpr (CPLX) {
                    ai[a] = xi[wm + a * 8 + (lane >> 2)][ka];
                    bi[a] = yi[wn + a * 8 + (lane >> 2)][ka];
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    dmma(cr[a][b][0], cr[a][b][1], ar[a], br[b]);
                    if constexpr (CPLX) {
                        dmma(cr[a][b][0], cr[a][b][1], ai[a], bi[b]);
                        dmma(ci[a][b][0], ci[a][b][1], ai[a], br[b]);
                        dmma(ci[a][b][0], ci[a][b][1], -ar[a], bi[b]);
                    }
                }
        }
        __syncthreads();
    }
    // accumulate into A_g (layout [G][n][n] x e doubles)
    const int e = CPLX ? 2 : 1;
    double *out = acc + (int64_t)g * n * n * e;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = i0 + wm + a * 8 + (lane >> 2);
                const int j = j0 + wn + b * 8 + (lane & 3) * 2 + h;
                if (i < n && j < n) {
                    double *p = out + ((int64_t)i * n + j) * e;
                    p[0] += cr[a][b][h];
                    if (CPLX) p[1] += ci[a][b][h];
                }
            }
}

}  // namespace

template <typename S>
void launch_contract(const S *x, const S *y, double *acc, int n, int ld, int chains, int gs, int T,
                     cudaStream_t st) {
    const int G = chains / gs;
    dim3 grid((n + BN - 1) / BN, (n + BM - 1) / BM, G);
    contract_kernel<S, ScalarTraits<S>::kDoubles == 2><<<grid, 128, 0, st>>>(x, y, acc, n, ld, gs, T);
}

template void launch_contract<double>(const double *, const double *, double *, int, int, int, int, int,
                                      cudaStream_t);
template void launch_contract<cd>(const cd *, const cd *, double *, int, int, int, int, int, cudaStream_t);

}  // namespace mcinv
