// sweep3.cu -- K1/K2 (v3): the CC sweep on the level schedule (levels.h),
// with fused accumulation.
//
// One CTA owns C consecutive chains (C a power of two) and runs all their
// sweeps with no grid synchronisation. A sweep is the sequence of phases
// 0..D: phase l updates every row of level l for the CTA's C chains at once
// (items = rows x chains, chain fastest, so the C lanes of a row read the same
// coefficients and gather C consecutive chains of row j: coalesced), then the
// CTA synchronises. The level schedule reads exactly the operands of the
// sequential row order of Eq. (4)/(5), so z and w are
// bit-identical to it:
//
//   z_i = sigma_i phi - delta_i * (sum_{j in U_i} a_ij z_j)                (Eq. 4)
//   w_i = conj(sigma_i) phi - conj(delta_i) * (sum_{j in U_i} b_ij w_j)    (Eq. 5)
//
// with the sums by serial fma from 0 in ascending j (reading R10)
// and phi = phi(chain, sweep, row) shared by z_i and w_i.
// Sampling sweeps accumulate (Eq. 1/C and Eq. tr): diag and the
// pattern pairs of row i with its lower neighbours at the update; deferred
// pattern pairs and the trace terms w_i^* Q_ij z_j as extra items of the
// phase after both values became final. Sums over the P = min(gs, C) chains
// of an accumulator sub-slot are warp shuffles; each sub-slot belongs to one
// CTA, so the slot updates are plain (deterministic) read-modify-writes.
#include "mcinv_internal.cuh"
#include "noise.cuh"
#include "scalar.cuh"

namespace mcinv {

namespace {

template <typename S>
__device__ __forceinline__ S seg_sum(S v, int P, unsigned mask) {
    for (int off = 1; off < P; off <<= 1) {
        if constexpr (ScalarTraits<S>::kDoubles == 1) {
            v += __shfl_xor_sync(mask, v, off);
        } else {
            v.re += __shfl_xor_sync(mask, v.re, off);
            v.im += __shfl_xor_sync(mask, v.im, off);
        }
    }
    return v;
}

template <typename S>
__device__ __forceinline__ ZW<S> ld_zw(const ZW<S> *p) {
    return *p;  // coherent load: values written by other threads of the CTA before __syncthreads
}

// fma chains of Eq. (4)/(5) over entries [beg, end), KU loads in flight
template <typename S, int KU>
__device__ __forceinline__ void row_sums(const Sweep3Params<S> &p, const ZW<S> *zcol, int beg, int end, S &az,
                                         S &aw) {
    for (int e0 = beg; e0 < end; e0 += KU) {
        int j[KU];
        ZW<S> v[KU];
        S a[KU], b[KU];
#pragma unroll
        for (int k = 0; k < KU; ++k)
            if (e0 + k < end) j[k] = __ldg(p.ent_col + e0 + k);
#pragma unroll
        for (int k = 0; k < KU; ++k)
            if (e0 + k < end) {
                v[k] = ld_zw(zcol + (int64_t)j[k] * p.ld);
                a[k] = ldg_s(p.ent_ab + 2 * (e0 + k));
                b[k] = ldg_s(p.ent_ab + 2 * (e0 + k) + 1);
            }
#pragma unroll
        for (int k = 0; k < KU; ++k)
            if (e0 + k < end) {
                az = fma_s(a[k], v[k].z, az);
                aw = fma_s(b[k], v[k].w, aw);
            }
    }
}

template <typename S>
__device__ __forceinline__ void slot_rmw(double *slot, S v) {
    add_to(slot, v);
}

}  // namespace

template <typename S, int KU, int NT>
__global__ void __launch_bounds__(NT, 1) sweep3_kernel(const Sweep3Params<S> p) {
    constexpr int E = ScalarTraits<S>::kDoubles;
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    const int lgC = p.lgC, lgP = p.lgP;
    const int C = 1 << lgC, P = 1 << lgP;
    const int c = tid & (C - 1);
    const int chain = (blockIdx.x << lgC) + c;
    const bool active = chain < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);
    const int lane = tid & 31;
    const unsigned pmask = P >= 32 ? 0xffffffffu : (((1u << P) - 1u) << (lane & ~(P - 1)));
    const bool pleader = (c & (P - 1)) == 0;
    const int64_t sub = chain >> lgP;  // accumulator sub-slot of this chain
    ZW<S> *__restrict__ zcol = p.zw + chain;
    const bool want_diag = p.outputs & OUT_DIAG, want_pat = p.outputs & OUT_PATTERN;
    const bool want_tr = p.outputs & OUT_TRACE, want_full = p.outputs & OUT_FULL;
    S tr = zero_s<S>();

    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const int nph = sampling ? p.D + 1 : p.D;
        for (int ph = 0; ph < nph; ++ph) {
            // ---- row updates of level ph
            const int r0 = __ldg(p.ph_row + ph);
            const int nu = (__ldg(p.ph_row + ph + 1) - r0) << lgC;
            for (int t = tid; t < nu; t += B) {
                const int o = r0 + (t >> lgC);
                const int i = __ldg(p.ord_row + o);
                const int beg = __ldg(p.ord_eptr + o), end = __ldg(p.ord_eptr + o + 1);
                double phi;
                if (p.noise == 0) phi = gaussian(static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
                else phi = p.noise == 2 ? 1.0 : 0.0;
                S az = zero_s<S>(), aw = zero_s<S>();
                row_sums<S, KU>(p, zcol, beg, end, az, aw);
                const S dl = ldg_s(p.ord_dsg + 2 * o), sg = ldg_s(p.ord_dsg + 2 * o + 1);
                const S zi = fma_s(neg_s(dl), az, scale_s(sg, phi));
                const S wi = fma_s(neg_s(conj_s(dl)), aw, scale_s(conj_s(sg), phi));
                zcol[(int64_t)i * p.ld] = ZW<S>{zi, wi};
                if (!sampling) continue;
                if (want_full) {
                    const int64_t ts = s - p.snap_s0;
                    p.snap_x[(ts * p.n + i) * p.ld + chain] = zi;
                    p.snap_y[(ts * p.n + i) * p.ld + chain] = wi;
                }
                if (want_diag || want_pat) {
                    const S d = seg_sum(active ? zwc_s(zi, wi) : zero_s<S>(), P, pmask);
                    if (pleader && active) {
                        if (want_diag) slot_rmw(p.slot_diag + (sub * p.n + i) * E, d);
                        if (want_pat) {
                            const int ps = __ldg(p.ord_pself + o);
                            if (ps >= 0) slot_rmw(p.slot_pat + (sub * p.pcount + ps) * E, d);
                        }
                    }
                }
                if (want_pat) {
                    // pairs with lower neighbours j: z_i w_j^* and z_j w_i^* (values final; L1-hot)
                    for (int e = beg; e < end; ++e) {
                        const int2 pz = __ldg(p.ent_pz + e);
                        if ((pz.x & pz.y) < 0) continue;  // both -1
                        const ZW<S> v = ld_zw(zcol + (int64_t)__ldg(p.ent_col + e) * p.ld);
                        if (pz.x >= 0) {
                            const S x = seg_sum(active ? zwc_s(zi, v.w) : zero_s<S>(), P, pmask);
                            if (pleader && active) slot_rmw(p.slot_pat + (sub * p.pcount + pz.x) * E, x);
                        }
                        if (pz.y >= 0) {
                            const S x = seg_sum(active ? zwc_s(v.z, wi) : zero_s<S>(), P, pmask);
                            if (pleader && active) slot_rmw(p.slot_pat + (sub * p.pcount + pz.y) * E, x);
                        }
                    }
                }
            }
            if (sampling) {
                // ---- deferred trace items: conj(w_i) sum_j Q_ij z_j  (w^dagger Q z, reading R2)
                if (want_tr) {
                    const int q0 = __ldg(p.ph_tq + ph);
                    const int nq = (__ldg(p.ph_tq + ph + 1) - q0) << lgC;
                    for (int t = tid; t < nq; t += B) {
                        const int o = q0 + (t >> lgC);
                        const int i = __ldg(p.tq_row + o);
                        S qz = zero_s<S>();
                        for (int e = __ldg(p.tq_eptr + o); e < __ldg(p.tq_eptr + o + 1); ++e)
                            qz = add_s(qz, mul_s(ldg_s(p.tq_val + e), ld_zw(zcol + (int64_t)__ldg(p.tq_col + e) * p.ld).z));
                        tr = add_s(tr, zwc_s(qz, ld_zw(zcol + (int64_t)i * p.ld).w));
                    }
                }
                // ---- deferred pattern pairs z_i w_j^*
                if (want_pat) {
                    const int q0 = __ldg(p.ph_pp + ph);
                    const int nq = (__ldg(p.ph_pp + ph + 1) - q0) << lgC;
                    for (int t = tid; t < nq; t += B) {
                        const int o = q0 + (t >> lgC);
                        const S zi = ld_zw(zcol + (int64_t)__ldg(p.pp_i + o) * p.ld).z;
                        const S wj = ld_zw(zcol + (int64_t)__ldg(p.pp_j + o) * p.ld).w;
                        const S x = seg_sum(active ? zwc_s(zi, wj) : zero_s<S>(), P, pmask);
                        if (pleader && active) slot_rmw(p.slot_pat + (sub * p.pcount + __ldg(p.pp_slot + o)) * E, x);
                    }
                }
            }
            __syncthreads();
        }
    }

    if (want_tr) {
        // per-chain trace: sum over the threads of each chain, then over the P chains of a sub-slot
        extern __shared__ __align__(16) unsigned char red_raw[];
        S *red = reinterpret_cast<S *>(red_raw);
        red[tid] = active ? tr : zero_s<S>();
        __syncthreads();
        if (tid < C) {
            S v = zero_s<S>();
            for (int h = tid; h < B; h += C) v = add_s(v, red[h]);
            const unsigned m = C >= 32 ? 0xffffffffu : ((1u << C) - 1u);
            const unsigned pm = P >= 32 ? m : (((1u << P) - 1u) << (lane & ~(P - 1)));
            v = seg_sum(v, P, pm);
            if (pleader && active) slot_rmw(p.slot_trace + sub * E, v);
        }
    }
}

template <typename S>
cudaError_t launch_sweep3(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    constexpr int KU = ScalarTraits<S>::kDoubles == 1 ? 4 : 2;
    const int C = 1 << p.lgC;
    const int blocks = (p.chains + C - 1) / C;
    const size_t smem = (p.outputs & OUT_TRACE) ? (size_t)threads * sizeof(S) : 0;
    // <= 512 threads: up to 128 registers, no spills; else 64 registers
    if (threads <= 512) sweep3_kernel<S, KU, 512><<<blocks, threads, smem, st>>>(p);
    else sweep3_kernel<S, KU, 1024><<<blocks, threads, smem, st>>>(p);
    return cudaGetLastError();
}

template cudaError_t launch_sweep3<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep3<cd>(const Sweep3Params<cd> &, int, cudaStream_t);

}  // namespace mcinv
