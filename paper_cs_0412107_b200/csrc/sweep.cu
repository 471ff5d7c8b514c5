// sweep.cu -- K1/K2: the CC sweep kernel with fused accumulation.
//
// One thread = one chain. Each thread walks rows i = 0..n-1 in the paper's
// sequential order (Eq. 4 and Eq. 5) for the sweeps of
// this launch, updating z_i and w_i in place in the [n][ld] state (chains
// contiguous, so every gather of row j is a coalesced warp load). No grid
// synchronisation: chains are independent.
//
//   z_i = sigma_i phi - delta_i * (sum_{j in U_i} a_ij z_j)         (Eq. 4)
//   w_i = conj(sigma_i) phi - conj(delta_i) * (sum b_ij w_j)        (Eq. 5)
//
// sums by serial fma from 0 in ascending j (reading R10). During sampling
// sweeps the estimators are accumulated at the row where both factors are
// final (K2): diag at row i, pattern (i,j) at row max(i,j), trace
// w^dagger Q z split by max(i,j) into registers (Eq. 1/C and Eq. tr,
// P:173-182).
#include "mcinv_internal.cuh"
#include "noise.cuh"
#include "scalar.cuh"

namespace mcinv {

template <typename S>
__device__ __forceinline__ S group_sum(S v, int gs) {
    for (int off = 1; off < gs; off <<= 1) v = add_s(v, shfl_xor_s(v, off));
    return v;
}

template <typename S>
__device__ __forceinline__ void slot_add(double *slot, int64_t idx, S v) {
    double *p = slot + idx * ScalarTraits<S>::kDoubles;
    add_to(p, v);
}

template <typename S>
__global__ void __launch_bounds__(128) sweep_kernel(const SweepParams<S> p) {
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;  // local chain (padded)
    if (c - lane >= p.ld) return;                            // whole warp beyond the padded range
    const bool active = c < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(c);
    const int n = p.A.n;
    const int ld = p.ld;
    ZW<S> *__restrict__ zw = p.zw;
    const bool leader = (lane & (p.gs - 1)) == 0;
    const int g = c / p.gs;
    S tr = zero_s<S>(), trs = zero_s<S>();  // trace over the launch / the current sweep
    bool dv = false;  // divergence seen (reading R12: every stored value is a sweep-end value)

    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        for (int i = 0; i < n; ++i) {
            const int beg = __ldg(p.A.u_ptr + i), end = __ldg(p.A.u_ptr + i + 1);
            S az = zero_s<S>(), aw = zero_s<S>();
            for (int e = beg; e < end; ++e) {
                const int j = __ldg(p.A.u_col + e);
                const ZW<S> v = zw[static_cast<int64_t>(j) * ld + c];
                az = fma_s(ldg_s(p.A.u_a + e), v.z, az);
                aw = fma_s(ldg_s(p.A.u_b + e), v.w, aw);
            }
            const double phi = noise_phi(p.noise, static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
            const S dl = ldg_s(p.A.delta + i), sg = ldg_s(p.A.sigma + i);
            const S zi = fma_s(neg_s(dl), az, scale_s(sg, phi));
            const S wi = fma_s(neg_s(conj_s(dl)), aw, scale_s(conj_s(sg), phi));
            zw[static_cast<int64_t>(i) * ld + c] = ZW<S>{zi, wi};
            dv = dv || bad_s(zi) || bad_s(wi);
            if (!sampling) continue;

            if (p.outputs & OUT_DIAG) {
                S v = active ? zwc_s(zi, wi) : zero_s<S>();
                v = group_sum(v, p.gs);
                if (leader && active) slot_add(p.slot_diag, static_cast<int64_t>(g) * n + i, v);
            }
            if (p.outputs & OUT_PATTERN) {
                const int pb = __ldg(p.P.p_ptr + i), pe = __ldg(p.P.p_ptr + i + 1);
                for (int q = pb; q < pe; ++q) {
                    const int code = __ldg(p.P.p_other + q);
                    const int o = code & 0x7fffffff;
                    S v;
                    if (o == i) {
                        v = zwc_s(zi, wi);
                    } else {
                        const ZW<S> u = zw[static_cast<int64_t>(o) * ld + c];
                        v = (code < 0) ? zwc_s(u.z, wi) : zwc_s(zi, u.w);
                    }
                    if (!active) v = zero_s<S>();
                    v = group_sum(v, p.gs);
                    if (leader && active)
                        slot_add(p.slot_pat, static_cast<int64_t>(g) * p.P.count + __ldg(p.P.p_idx + q), v);
                }
            }
            if (p.outputs & OUT_TRACE) {
                S qz = zero_s<S>();
                for (int q = __ldg(p.Q.qr_ptr + i); q < __ldg(p.Q.qr_ptr + i + 1); ++q) {
                    const int j = __ldg(p.Q.qr_col + q);
                    const S zj = (j == i) ? zi : zw[static_cast<int64_t>(j) * ld + c].z;
                    qz = add_s(qz, mul_s(ldg_s(p.Q.qr_val + q), zj));
                }
                S qw = zero_s<S>();
                for (int q = __ldg(p.Q.qc_ptr + i); q < __ldg(p.Q.qc_ptr + i + 1); ++q) {
                    const int r = __ldg(p.Q.qc_row + q);
                    qw = add_s(qw, mul_s(ldg_s(p.Q.qc_val + q), conj_s(zw[static_cast<int64_t>(r) * ld + c].w)));
                }
                trs = add_s(trs, add_s(zwc_s(qz, wi), mul_s(zi, qw)));
            }
            if (p.outputs & OUT_FULL) {
                const int64_t t = s - p.snap_s0;
                p.snap_x[(t * n + i) * ld + c] = zi;
                p.snap_y[(t * n + i) * ld + c] = wi;
            }
        }
        if ((p.outputs & OUT_TRACE) && sampling) {
            if (p.series) {  // the sweep's realized trace of this warp's chains (Geyer's series)
                S v = active ? trs : zero_s<S>();
                v = group_sum(v, 32);
                if (lane == 0) atomic_add_to(p.series + (int64_t)(p.series_base + s - p.burn_in) * ScalarTraits<S>::kDoubles, v);
            }
            tr = add_s(tr, trs);
            trs = zero_s<S>();
        }
    }
    if (p.outputs & OUT_TRACE) {
        S v = active ? tr : zero_s<S>();
        v = group_sum(v, p.gs);
        if (leader && active) slot_add(p.slot_trace, g, v);
    }
    if (dv && active) atomicAdd(p.bad, 1.0);
}

template <typename S>
void launch_sweep(const SweepParams<S> &p, cudaStream_t st) {
    // Few chains per GPU (BASELINE configs: 64-16384): spread warps over all
    // SMs first, one warp per CTA until the grid exceeds the SM count.
    const int warps = p.ld / 32;
    const int wpb = warps >= 4 * 148 ? 4 : (warps >= 2 * 148 ? 2 : 1);
    const int threads = 32 * wpb;
    const int blocks = (p.ld + threads - 1) / threads;
    sweep_kernel<S><<<blocks, threads, 0, st>>>(p);
}

template void launch_sweep<double>(const SweepParams<double> &, cudaStream_t);
template void launch_sweep<cd>(const SweepParams<cd> &, cudaStream_t);

}  // namespace mcinv
