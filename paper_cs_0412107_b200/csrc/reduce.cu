// reduce.cu -- K4: group moments, finalize (estimate + standard error),
// the coupled-burn-in reduction, and the test-only Philox/Gaussian dump kernels.
//
// Estimate (Eq. 1/C):  est = S1 / (m (M-N)).
// Standard error (reading R15, replacing the Geyer error of
// P:354-360): group means mu_g = S_g / (gs (M-N)); SE = sd(mu_g) / sqrt(G).
#include "mcinv_internal.cuh"
#include "noise.cuh"
#include "scalar.cuh"

namespace mcinv {

// slot layout [G * k][comps]: the sum of group g is the sum of its k sub-slots.
// s1[c] = sum_g (group sum g); m2[c] = sum_g (group sum - mean)^2, two-pass about the
// mean of these G groups (no cancellation of a raw sum of squares). With `center`
// (after a cross-rank all-reduce of s1): s1 is left alone and m2 is taken about the
// global mean center[c] / center_G instead, so that a SUM of the ranks' m2 is the
// scatter of all groups about the global mean (mcinv_recenter).
__global__ void moments_kernel(const double *__restrict__ slot, int G, int k, int64_t comps,
                               double *__restrict__ s1, double *__restrict__ m2,
                               const double *__restrict__ center, double center_G) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < comps;
         c += (int64_t)gridDim.x * blockDim.x) {
        double mean;
        if (center) {
            mean = center[c] / center_G;
        } else {
            double a = 0.0;
            for (int g = 0; g < G; ++g) {
                double v = 0.0;
                for (int h = 0; h < k; ++h) v += slot[((int64_t)g * k + h) * comps + c];
                a += v;
            }
            s1[c] = a;
            mean = a / (double)G;
        }
        double b = 0.0;
        for (int g = 0; g < G; ++g) {
            double v = 0.0;
            for (int h = 0; h < k; ++h) v += slot[((int64_t)g * k + h) * comps + c];
            const double d = v - mean;
            b = fma(d, d, b);
        }
        m2[c] = b;
    }
}

// estimate = S1 / (m (M-N)); SE = sqrt(var(group means) / G) with
// var(group means) = M2 / ((gs (M-N))^2 (G - 1))  (reading R15)
__global__ void finalize_kernel(const double *__restrict__ s1, const double *__restrict__ m2, int64_t comps,
                                double m_cycles, double gs_cycles, double G, double *__restrict__ est,
                                double *__restrict__ se) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < comps;
         c += (int64_t)gridDim.x * blockDim.x) {
        est[c] = s1[c] / m_cycles;
        if (se) {
            const double var = G > 1.0 ? m2[c] / (gs_cycles * gs_cycles * (G - 1.0)) : NAN;
            se[c] = sqrt(var / G);
        }
    }
}

// max over rows of the (z, w) moduli of chain 0 (the coupled-burn-in difference)
template <typename S>
__global__ void max_modulus_kernel(const ZW<S> *__restrict__ zw, int n, int ld, double *out) {
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const ZW<S> v = zw[(int64_t)i * ld];
        double a, b;
        if constexpr (ScalarTraits<S>::kDoubles == 1) {
            a = fabs(v.z);
            b = fabs(v.w);
        } else {
            a = hypot(v.z.re, v.z.im);
            b = hypot(v.w.re, v.w.im);
        }
        m = fmax(m, fmax(a, b));
        if (!(a <= 1e300) || !(b <= 1e300)) m = INFINITY;  // non-finite: diverged
    }
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    __shared__ double part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) r = fmax(r, part[w]);
        *out = r;
    }
}

template <typename S>
void launch_max_modulus(const ZW<S> *zw, int n, int ld, double *out, cudaStream_t st) {
    max_modulus_kernel<S><<<1, 1024, 0, st>>>(zw, n, ld, out);
}
template void launch_max_modulus<double>(const ZW<double> *, int, int, double *, cudaStream_t);
template void launch_max_modulus<cd>(const ZW<cd> *, int, int, double *, cudaStream_t);

__global__ void philox_kernel(const uint32_t *__restrict__ ctr, int64_t count, uint32_t k0, uint32_t k1,
                              uint32_t *__restrict__ out, double *__restrict__ gauss) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
         t += (int64_t)gridDim.x * blockDim.x) {
        const PhiloxOut r = philox4x32_10(ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], ctr[4 * t + 3], k0, k1);
        if (out) {
            out[4 * t] = r.x;
            out[4 * t + 1] = r.y;
            out[4 * t + 2] = r.z;
            out[4 * t + 3] = r.w;
        }
        // the kernels' noise of (row, sweep, chain) = (ctr[0], ctr[1], ctr[2]) (reading R4)
        if (gauss) gauss[t] = gaussian(ctr[4 * t], ctr[4 * t + 1], ctr[4 * t + 2], k0, k1);
    }
}

static int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    return b < 1 ? 1 : (int)b;
}

void launch_moments(const double *slot, int G, int k, int64_t comps, double *s1, double *m2, const double *center,
                    double center_G, cudaStream_t st) {
    moments_kernel<<<grid_for(comps, 256), 256, 0, st>>>(slot, G, k, comps, s1, m2, center, center_G);
}

void launch_finalize(const double *s1, const double *m2, int64_t comps, double m_cycles, double gs_cycles, double G,
                     double *est, double *se, cudaStream_t st) {
    finalize_kernel<<<grid_for(comps, 256), 256, 0, st>>>(s1, m2, comps, m_cycles, gs_cycles, G, est, se);
}

// Geyer's initial positive sequence estimator (Geyer 1992; the paper's standard errors,
// PAPER.md:354-360) of component c = blockIdx.x of the series x[t * e + c], t < m: mean,
// lag-k autocovariances gamma_k = (1/m) sum_t (x_t - mean)(x_{t+k} - mean) (each summed in
// t order by one thread, a batch of 1024 lags at a time), pair sums gamma_2j + gamma_2j+1
// while positive, sigma2 = -gamma_0 + 2 sum, ESS = m gamma_0 / sigma2.
__global__ void geyer_kernel(const double *__restrict__ x, int64_t m, int e, double *__restrict__ out) {
    const int c = blockIdx.x;
    __shared__ double gam[1024 + 1];
    __shared__ double s_mean, s_sigma2;
    __shared__ int s_done;
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int64_t t = 0; t < m; ++t) a += x[t * e + c];
        s_mean = a / (double)m;
        s_sigma2 = 0.0;
        s_done = 0;
    }
    __syncthreads();
    const double mean = s_mean;
    double g0 = 0.0;
    for (int64_t l0 = 0; !s_done; l0 += 1024) {
        const int64_t lag = l0 + threadIdx.x;
        double acc = 0.0;
        if (lag < m)
            for (int64_t t = 0; t + lag < m; ++t) acc += (x[t * e + c] - mean) * (x[(t + lag) * e + c] - mean);
        gam[threadIdx.x] = acc / (double)m;
        __syncthreads();
        if (threadIdx.x == 0) {
            if (l0 == 0) {
                g0 = gam[0];
                s_sigma2 = -g0;
                gam[1024] = g0;
            }
            for (int q = 0; q < 1024; q += 2) {
                const int64_t j2 = l0 + q;  // pair (j2, j2 + 1)
                if (j2 + 1 >= m || !(gam[q] + gam[q + 1] > 0.0)) {
                    s_done = 1;
                    break;
                }
                s_sigma2 += 2.0 * (gam[q] + gam[q + 1]);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double gg0 = gam[1024];
        out[4 * c] = mean;
        out[4 * c + 1] = gg0;
        out[4 * c + 2] = s_sigma2;
        out[4 * c + 3] = s_sigma2 > 0.0 ? (double)m * gg0 / s_sigma2 : 0.0;
    }
}

void launch_geyer(const double *x, int64_t m, int e, double *out, cudaStream_t st) {
    geyer_kernel<<<e, 1024, 0, st>>>(x, m, e, out);
}

void launch_philox(const uint32_t *ctr, int64_t count, uint32_t k0, uint32_t k1, uint32_t *out, double *gauss,
                   cudaStream_t st) {
    philox_kernel<<<grid_for(count, 256), 256, 0, st>>>(ctr, count, k0, k1, out, gauss);
}

}  // namespace mcinv
