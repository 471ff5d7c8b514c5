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
        if (gauss) gauss[t] = box_muller(r);
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

void launch_philox(const uint32_t *ctr, int64_t count, uint32_t k0, uint32_t k1, uint32_t *out, double *gauss,
                   cudaStream_t st) {
    philox_kernel<<<grid_for(count, 256), 256, 0, st>>>(ctr, count, k0, k1, out, gauss);
}

}  // namespace mcinv
