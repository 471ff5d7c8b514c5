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
//
// Sampling sweeps accumulate (Eq. 1/C and Eq. tr): at row i's
// update the products z_i w_i^* (diag, and the pattern element (i,i)) and,
// for every lower neighbour j (a prefix of the ascending entry list, values
// final), z_i w_j^* and z_j w_i^*; other pattern pairs and the trace terms
// w_i^* Q_ij z_j are deferred items of the phase after both values became
// final. The P lanes of one SE group (P = min(group size, C), a template
// parameter) sum their products with a transpose-reduction (V = min(P, 8)
// products over P lanes in V-1 shuffles, then log2(P/V) butterflies), after
// which each lane posts ONE fire-and-forget reduction (red.global.add) into
// the group's slot; the slots of all groups (41 MB for config 2) stay in L2.
#include <cstdlib>

#include "sweep_common.cuh"

namespace mcinv {


// GAUSS: compile-time Gaussian noise (the default mode; +2.4% config 4, +1.1% config 5)
template <typename S, int KU, int NT, int LGP, int K, bool GAUSS = false>
__global__ void __launch_bounds__(NT, 1) sweep3_kernel(const Sweep3Params<S> p) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    constexpr int E = ScalarTraits<S>::kDoubles;
    constexpr int P = 1 << LGP;        // lanes of one SE group inside this CTA (K chains per lane)
    constexpr int V = P < 8 ? P : 8;   // products per transpose-reduction (pairs of one entry)
    const int tid = threadIdx.x;
    const int B = blockDim.x;  // a multiple of 32 and of C / K
    const int lane = tid & 31;
    const int wbase = tid - lane;
    const int lgL = p.lgC - (K == 2 ? 1 : 0);  // log2 lanes per row: C / K
    const int Lr = 1 << lgL;
    const int cl = tid & (Lr - 1);
    const int chain = (blockIdx.x << p.lgC) + cl * K;  // first of this lane's K chains
    bool active[K];
#pragma unroll
    for (int h = 0; h < K; ++h) active[h] = chain + h < p.chains;
    const bool gleader = (cl & (P - 1)) == 0;                     // owner of a plain group sum
    const bool towner = (lane & ((P > V ? P / V : 1) - 1)) == 0;  // owner of a transposed value
    const int64_t grp = chain >> p.lgG;  // SE group of these chains = their accumulator slot
    ZW<S> *__restrict__ zcol = p.zw + chain;
    const bool want_diag = p.outputs & OUT_DIAG, want_pat = p.outputs & OUT_PATTERN;
    const bool want_tr = p.outputs & OUT_TRACE, want_full = p.outputs & OUT_FULL;
    double *const sd = p.slot_diag + grp * p.n * E;
    double *const sp = p.slot_pat + grp * p.pcount * E;
    S tr = zero_s<S>();   // K == 1 only (trace runs use K = 1): the chain's trace over the launch
    S trs = zero_s<S>();  // ... and over the current sweep (Geyer's series)
    bool dv = false;     // divergence seen (reading R12)

    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const int nph = sampling ? p.D + 1 : p.D;
        for (int ph = 0; ph < nph; ++ph) {
            // ---- row updates of level ph; warp-uniform trip count (shuffles below)
            const int r0 = __ldg(p.ph_row + ph);
            const int nu = (__ldg(p.ph_row + ph + 1) - r0) << lgL;
            for (int base = wbase; base < nu; base += B) {
                const int t = base + lane;
                const bool valid = t < nu;
                const int o = r0 + (t >> lgL);
                const int4 rec = valid ? __ldg(p.ord_rec + o) : make_int4(0, 0, 0, -1);
                const int i = rec.x, beg = rec.y, cnt = rec.z & 0xffff;
                S zi[K], wi[K];
#pragma unroll
                for (int h = 0; h < K; ++h) zi[h] = wi[h] = zero_s<S>();
                if (valid) {
                    if (p.prefetch == 3)  // the neighbours' state lines into L2 while the noise runs
                        for (int e = 0; e < cnt; ++e) prefetch_l2(zrow(zcol, __ldg(p.ent_col + beg + e), zst));
                    // noise first: its temporaries are dead before the gathers are in flight
                    double phi[K];
                    if constexpr (GAUSS && K == 2) {
                        // the thread's chains are a Box-Muller pair (2m, 2m + 1; reading R4): one
                        // Philox block, one ln and sqrt for both
                        gaussian2(static_cast<uint32_t>(i), k, p.chain0 + static_cast<uint32_t>(chain), p.key0, p.key1,
                                  phi[0], phi[K - 1]);
                    } else {
#pragma unroll
                        for (int h = 0; h < K; ++h) {
                            if constexpr (GAUSS)
                                phi[h] = gaussian(static_cast<uint32_t>(i), k,
                                                  p.chain0 + static_cast<uint32_t>(chain + h), p.key0, p.key1);
                            else
                                phi[h] = noise_phi(p.noise, static_cast<uint32_t>(i), k,
                                                   p.chain0 + static_cast<uint32_t>(chain + h), p.key0, p.key1);
                        }
                    }
                    S az[K], aw[K];
#pragma unroll
                    for (int h = 0; h < K; ++h) az[h] = aw[h] = zero_s<S>();
                    row_sums<S, KU, K>(p, zcol, beg, cnt, az, aw);
                    const S dl = ldg_s(p.ord_dsg + 2 * o), sg = ldg_s(p.ord_dsg + 2 * o + 1);
                    ZWK<S, K> out;
#pragma unroll
                    for (int h = 0; h < K; ++h) {
                        zi[h] = fma_s(neg_s(dl), az[h], scale_s(sg, phi[h]));
                        wi[h] = fma_s(neg_s(conj_s(dl)), aw[h], scale_s(conj_s(sg), phi[h]));
                        out.v[h] = ZW<S>{zi[h], wi[h]};
                    }
                    st_zwk<S, K>(zrow(zcol, i, zst), out);
#pragma unroll
                    for (int h = 0; h < K; ++h) dv = dv | (active[h] & (bad_s(zi[h]) | bad_s(wi[h])));
                    if (want_full && sampling) {
                        const int64_t ts = s - p.snap_s0;
#pragma unroll
                        for (int h = 0; h < K; ++h) {
                            p.snap_x[(ts * p.n + i) * p.ld + chain + h] = zi[h];
                            p.snap_y[(ts * p.n + i) * p.ld + chain + h] = wi[h];
                        }
                    }
                }
                if (!sampling) continue;
                bool acc[K];
#pragma unroll
                for (int h = 0; h < K; ++h) acc[h] = valid && active[h];
                accumulate_row<S, P, V, K>(p, zcol, rec, zi, wi, acc, lane, gleader, towner, sd, sp, want_diag,
                                           want_pat);
            }
            if constexpr (K == 1) {
                if (sampling) {
                    // ---- deferred trace items: conj(w_i) sum_j Q_ij z_j  (w^dagger Q z, reading R2);
                    // per-thread register sums, no shuffles
                    if (want_tr) {
                        const int q0 = __ldg(p.ph_tq + ph);
                        const int nq = (__ldg(p.ph_tq + ph + 1) - q0) << lgL;
                        for (int t = tid; t < nq; t += B) {
                            const int o = q0 + (t >> lgL);
                            const int i = __ldg(p.tq_row + o);
                            S qz = zero_s<S>();
                            for (int e = __ldg(p.tq_eptr + o); e < __ldg(p.tq_eptr + o + 1); ++e)
                                qz = add_s(qz, mul_s(ldg_s(p.tq_val + e),
                                                     ld_zw(zrow(zcol, __ldg(p.tq_col + e), zst)).z));
                            trs = add_s(trs, zwc_s(qz, ld_zw(zrow(zcol, i, zst)).w));
                        }
                    }
                    // ---- deferred pattern pairs z_i w_j^*
                    if (want_pat) {
                        const int q0 = __ldg(p.ph_pp + ph);
                        const int nq = (__ldg(p.ph_pp + ph + 1) - q0) << lgL;
                        for (int base = wbase; base < nq; base += B) {
                            const int t = base + lane;
                            const bool valid = t < nq;
                            const int o = q0 + (t >> lgL);
                            S x = zero_s<S>();
                            if (valid && active[0])
                                x = zwc_s(ld_zw(zrow(zcol, __ldg(p.pp_i + o), zst)).z,
                                          ld_zw(zrow(zcol, __ldg(p.pp_j + o), zst)).w);
                            x = group_sum<P>(x);
                            if (valid && active[0] && gleader)
                                slot_red(sp + (int64_t)__ldg(p.pp_slot + o) * E, x);
                        }
                    }
                }
            }
            __syncthreads();
        }
        if constexpr (K == 1) {
            if (want_tr && sampling) {
                // the sweep's realized trace of this warp's chains into Geyer's series
                if (p.series) {
                    const S v = group_sum<32>(active[0] ? trs : zero_s<S>());
                    if (lane == 0) slot_red(p.series + (int64_t)(p.series_base + s - p.burn_in) * E, v);
                }
                tr = add_s(tr, trs);
                trs = zero_s<S>();
            }
        }
    }

    if (dv) atomicAdd(p.bad, 1.0);
    if constexpr (K == 1) {
        if (want_tr) {
            // per-chain trace: sum over the threads of each chain, then over the P chains of a group
            extern __shared__ __align__(16) unsigned char red_raw[];
            S *red = reinterpret_cast<S *>(red_raw);
            const int C = 1 << p.lgC;
            red[tid] = active[0] ? tr : zero_s<S>();
            __syncthreads();
            if (wbase < C) {  // whole warps (C < 32: lanes >= C hold zeros and are not leaders)
                S v = zero_s<S>();
                if (tid < C)
                    for (int h = tid; h < B; h += C) v = add_s(v, red[h]);
                v = group_sum<P>(v);
                if (tid < C && gleader && active[0]) slot_red(p.slot_trace + grp * E, v);
            }
        }
    }
}

// ---------------------------------------------------------------- v4: dataflow
//
// The same row update and accumulation, without per-level barriers: one CTA
// barrier per sweep, and within a sweep every row j has a completion counter
// done[j] (shared memory, one byte, counted modulo 256) = the number of
// sweeps that have updated it. Row i in sweep s may run once every lower
// neighbour j < i (a prefix of its ascending entry list) has done[j] = s + 1:
// it then reads their new values (Eq. 4/5 order). Upper neighbours hold their
// sweep s - 1 values until the sweep barrier (they are updated after row i in
// every order the counters allow, being at higher levels), and every read of
// row i's sweep s - 1 value happened before that barrier, so the sweep
// barrier covers all write-after-read hazards; the counter is published right
// after the store. Each warp takes groups of R = 32 / C rows (never spanning
// a level: rows of a group are independent) in level order; every dependency
// points to an earlier group, so the earliest unfinished group can always
// run: no deadlock. A bounded wait (watchdog) reports instead of hanging if
// that reasoning were ever violated.
template <typename S, int KU, int NT, int LGP, int K>
__global__ void __launch_bounds__(NT, 1) sweep4_kernel(const Sweep3Params<S> p) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    constexpr int E = ScalarTraits<S>::kDoubles;
    constexpr int P = 1 << LGP;        // lanes of one SE group (K chains per lane)
    constexpr int V = P < 8 ? P : 8;
    extern __shared__ __align__(16) unsigned char done[];  // [n]
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    const int lane = tid & 31;
    const int lgL = p.lgC - (K == 2 ? 1 : 0);  // log2 lanes per row (C / K <= 32: one warp)
    const int Lr = 1 << lgL;
    const int cl = lane & (Lr - 1);
    const int chain = (blockIdx.x << p.lgC) + cl * K;
    bool active[K];
#pragma unroll
    for (int h = 0; h < K; ++h) active[h] = chain + h < p.chains;
    const bool gleader = (cl & (P - 1)) == 0;
    const bool towner = (lane & ((P > V ? P / V : 1) - 1)) == 0;
    const int64_t grp = chain >> p.lgG;
    ZW<S> *__restrict__ zcol = p.zw + chain;
    const bool want_diag = p.outputs & OUT_DIAG, want_pat = p.outputs & OUT_PATTERN;
    const bool want_full = p.outputs & OUT_FULL;
    double *const sd = p.slot_diag + grp * p.n * E;
    double *const sp = p.slot_pat + grp * p.pcount * E;

    for (int j = tid; j < p.n; j += B) done[j] = static_cast<unsigned char>(p.s_begin);
    __syncthreads();
    bool dv = false;  // divergence seen (reading R12)

    const int R = 32 >> lgL;  // rows per warp group
    const int ngroups = p.nslots / R;
    const int W = B >> 5;
    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const unsigned char need = static_cast<unsigned char>(s + 1);
        // the next group's record is loaded one item ahead (off the item's critical path)
        int4 rec_next = (tid >> 5) < ngroups ? __ldg(p.slot_rec + (tid >> 5) * R + (lane >> lgL))
                                             : make_int4(-1, 0, 0, -1);
        for (int g = tid >> 5; g < ngroups; g += W) {
            const int slot = g * R + (lane >> lgL);
            const int4 rec = rec_next;
            if (g + W < ngroups) rec_next = __ldg(p.slot_rec + (g + W) * R + (lane >> lgL));
            const bool valid = rec.x >= 0;
            const int i = rec.x, beg = rec.y, cnt = valid ? rec.z & 0xffff : 0;
            S zi[K], wi[K];
#pragma unroll
            for (int h = 0; h < K; ++h) zi[h] = wi[h] = zero_s<S>();
            if (valid) {
                double phi[K];
#pragma unroll
                for (int h = 0; h < K; ++h) {
                    phi[h] = noise_phi(p.noise, static_cast<uint32_t>(i), k,
                                       p.chain0 + static_cast<uint32_t>(chain + h), p.key0, p.key1);
                }
                // wait for the lower neighbours (the first nlow entries; all lanes of the
                // row read the same counters: smem broadcast), then acquire
                const int nlow = static_cast<int>(static_cast<unsigned>(rec.z) >> 16);
                for (int e = 0; e < nlow; ++e) {
                    const volatile unsigned char *f = done + __ldg(p.ent_col + beg + e);
                    wait_ready([&] { return *f == need; }, p.err, p.spin_ns);
                }
                __threadfence_block();
                S az[K], aw[K];
#pragma unroll
                for (int h = 0; h < K; ++h) az[h] = aw[h] = zero_s<S>();
                row_sums<S, KU, K>(p, zcol, beg, cnt, az, aw);
                const S dl = ldg_s(p.slot_dsg + 2 * slot), sg = ldg_s(p.slot_dsg + 2 * slot + 1);
                ZWK<S, K> out;
#pragma unroll
                for (int h = 0; h < K; ++h) {
                    zi[h] = fma_s(neg_s(dl), az[h], scale_s(sg, phi[h]));
                    wi[h] = fma_s(neg_s(conj_s(dl)), aw[h], scale_s(conj_s(sg), phi[h]));
                    out.v[h] = ZW<S>{zi[h], wi[h]};
                }
                st_zwk<S, K>(zrow(zcol, i, zst), out);
#pragma unroll
                for (int h = 0; h < K; ++h) dv = dv | (active[h] & (bad_s(zi[h]) | bad_s(wi[h])));
                if (want_full && sampling) {
                    const int64_t ts = s - p.snap_s0;
#pragma unroll
                    for (int h = 0; h < K; ++h) {
                        p.snap_x[(ts * p.n + i) * p.ld + chain + h] = zi[h];
                        p.snap_y[(ts * p.n + i) * p.ld + chain + h] = wi[h];
                    }
                }
            }
            __syncwarp();  // the row's stores are ordered before its counter update
            if (valid && cl == 0) {
                __threadfence_block();  // release
                *reinterpret_cast<volatile unsigned char *>(done + i) = need;
            }
            if (sampling) {
                bool acc[K];
#pragma unroll
                for (int h = 0; h < K; ++h) acc[h] = valid && active[h];
                accumulate_row<S, P, V, K>(p, zcol, rec, zi, wi, acc, lane, gleader, towner, sd, sp, want_diag,
                                           want_pat);
            }
            if (p.reconv & 1) __syncwarp();  // reconverge before the next item (see v5)
        }
        __syncthreads();  // sweep boundary: all reads of sweep s values are done
    }
    if (dv) atomicAdd(p.bad, 1.0);
}

namespace {

template <typename S, int LGP, int K>
cudaError_t launch3k(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    // gathers in flight per row chunk: 64 registers at 1024 threads, 85 at 768, 128 at 512
    // (the entry arrays are padded by 8 entries: KU <= 8)
    constexpr int KS = ScalarTraits<S>::kDoubles == 1 && K == 1 ? 4 : 2;
    const int C = 1 << p.lgC;
    const int blocks = (p.chains + C - 1) / C;
    const size_t smem = (p.outputs & OUT_TRACE) ? (size_t)threads * sizeof(S) : 0;
    if (threads <= 512) sweep3_kernel<S, 2 * KS, 512, LGP, K><<<blocks, threads, smem, st>>>(p);
    else if (threads <= 768) sweep3_kernel<S, KS, 768, LGP, K><<<blocks, threads, smem, st>>>(p);
    else if (p.noise == 0) sweep3_kernel<S, KS, 1024, LGP, K, true><<<blocks, threads, smem, st>>>(p);
    else sweep3_kernel<S, KS, 1024, LGP, K><<<blocks, threads, smem, st>>>(p);
    return cudaGetLastError();
}

template <typename S, int LGP>
cudaError_t launch3(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    if constexpr (ScalarTraits<S>::kDoubles == 1) {
        if (p.lgK == 1) return launch3k<S, LGP, 2>(p, threads, st);
    }
    return launch3k<S, LGP, 1>(p, threads, st);
}

}  // namespace

template <typename S, int LGP, int K>
cudaError_t launch4k(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    constexpr int KS = ScalarTraits<S>::kDoubles == 1 && K == 1 ? 4 : 2;
    const int C = 1 << p.lgC;
    const int blocks = (p.chains + C - 1) / C;
    const size_t smem = ((size_t)p.n + 15) / 16 * 16;
    // shared memory only holds the counters: give the rest of the unified L1 to the cache
    // (plan data and the partner re-reads of the accumulation hit there)
    int carve = (int)((smem + 8192) * 100 / (228 * 1024)) + 1;
    if (const char *ev = std::getenv("MCINV_CARVE")) carve = std::atoi(ev);
    if (carve > 100) carve = 100;
    cudaError_t e;
    if (threads <= 512) {
        auto k = sweep4_kernel<S, 2 * KS, 512, LGP, K>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        if (e == cudaSuccess) k<<<blocks, threads, smem, st>>>(p);
    } else if (threads <= 768) {
        auto k = sweep4_kernel<S, KS, 768, LGP, K>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        if (e == cudaSuccess) k<<<blocks, threads, smem, st>>>(p);
    } else {
        auto k = sweep4_kernel<S, KS, 1024, LGP, K>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        if (e == cudaSuccess) k<<<blocks, threads, smem, st>>>(p);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename S, int LGP>
cudaError_t launch4(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    if constexpr (ScalarTraits<S>::kDoubles == 1) {
        if (p.lgK == 1) return launch4k<S, LGP, 2>(p, threads, st);
    }
    return launch4k<S, LGP, 1>(p, threads, st);
}

template <typename S>
cudaError_t launch_sweep4(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    switch (p.lgP) {
        case 0: return launch4<S, 0>(p, threads, st);
        case 1: return launch4<S, 1>(p, threads, st);
        case 2: return launch4<S, 2>(p, threads, st);
        case 3: return launch4<S, 3>(p, threads, st);
        case 4: return launch4<S, 4>(p, threads, st);
        case 5: return launch4<S, 5>(p, threads, st);
        default: return cudaErrorInvalidValue;
    }
}

template <typename S>
cudaError_t launch_sweep3(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    switch (p.lgP) {
        case 0: return launch3<S, 0>(p, threads, st);
        case 1: return launch3<S, 1>(p, threads, st);
        case 2: return launch3<S, 2>(p, threads, st);
        case 3: return launch3<S, 3>(p, threads, st);
        case 4: return launch3<S, 4>(p, threads, st);
        case 5: return launch3<S, 5>(p, threads, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_sweep3<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep3<cd>(const Sweep3Params<cd> &, int, cudaStream_t);
template cudaError_t launch_sweep4<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep4<cd>(const Sweep3Params<cd> &, int, cudaStream_t);

}  // namespace mcinv
