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
#include "mcinv_internal.cuh"
#include "noise.cuh"
#include "scalar.cuh"

namespace mcinv {

namespace {

__device__ __forceinline__ double shfl_x(double v, int off) { return __shfl_xor_sync(0xffffffffu, v, off); }
__device__ __forceinline__ cd shfl_x(cd v, int off) { return cd{shfl_x(v.re, off), shfl_x(v.im, off)}; }
__device__ __forceinline__ double sel(bool c, double a, double b) { return c ? a : b; }
__device__ __forceinline__ cd sel(bool c, cd a, cd b) { return cd{c ? a.re : b.re, c ? a.im : b.im}; }

// Sum over the P lanes of each aligned lane group (converged warp, full mask).
template <int P, typename S>
__device__ __forceinline__ S group_sum(S v) {
#pragma unroll
    for (int off = 1; off < P; off <<= 1) v = add_s(v, shfl_x(v, off));
    return v;
}

// Transpose-reduction of V values per lane over the P lanes of a group
// (V <= P, both powers of two). On return the lane holds the group total of
// value index `held`; P/V lanes hold each index, the one with
// (lane & (P/V - 1)) == 0 is its owner.
template <int P, int V, typename S>
__device__ __forceinline__ S transpose_sum(S (&v)[V], int lane, int &held) {
    held = 0;
    int nv = V;
#pragma unroll
    for (int off = P / 2; off >= 1; off >>= 1) {
        if (nv > 1) {
            const bool up = (lane & off) != 0;  // this lane keeps the upper half
#pragma unroll
            for (int q = 0; q < V / 2; ++q) {
                if (q < nv / 2) {
                    const S send = sel(up, v[q], v[q + nv / 2]);
                    const S keep = sel(up, v[q + nv / 2], v[q]);
                    v[q] = add_s(keep, shfl_x(send, off));
                }
            }
            if (up) held += nv / 2;
            nv /= 2;
        } else {
            v[0] = add_s(v[0], shfl_x(v[0], off));
        }
    }
    return v[0];
}

// the (a, b) coefficient pair of an entry in one (real) or two (complex) 16-B loads
__device__ __forceinline__ ZW<double> ldg_ab(const ZW<double> *p) {
    const double2 v = __ldg(reinterpret_cast<const double2 *>(p));
    return ZW<double>{v.x, v.y};
}
__device__ __forceinline__ ZW<cd> ldg_ab(const ZW<cd> *p) {
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    const double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    return ZW<cd>{cd{a.x, a.y}, cd{b.x, b.y}};
}

template <typename S>
__device__ __forceinline__ ZW<S> ld_zw(const ZW<S> *p) {
    return *p;  // coherent load: values written by other threads of the CTA before __syncthreads
}

// fma chains of Eq. (4)/(5) over the cnt entries at beg, KU gathers in flight.
// Branch-free: the entry arrays are padded by KU entries, so every load is
// unconditional; slots past the row's end gather row 0 of this chain (an
// L1-hot dummy) and their fma is predicated off, so the sums are exactly the
// serial ones.
template <typename S, int KU>
__device__ __forceinline__ void row_sums(const Sweep3Params<S> &p, const ZW<S> *zcol, int beg, int cnt, S &az,
                                         S &aw) {
    for (int e0 = 0; e0 < cnt; e0 += KU) {
        int j[KU];
        ZW<S> v[KU], ab[KU];
#pragma unroll
        for (int k = 0; k < KU; ++k) j[k] = __ldg(p.ent_col + beg + e0 + k);
#pragma unroll
        for (int k = 0; k < KU; ++k) {
            v[k] = ld_zw(zcol + (int64_t)(e0 + k < cnt ? j[k] : 0) * p.ld);
            ab[k] = ldg_ab(reinterpret_cast<const ZW<S> *>(p.ent_ab) + beg + e0 + k);
        }
#pragma unroll
        for (int k = 0; k < KU; ++k)
            if (e0 + k < cnt) {
                az = fma_s(ab[k].z, v[k].z, az);
                aw = fma_s(ab[k].w, v[k].w, aw);
            }
    }
}

__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void slot_red(double *slot, double v) { red_add(slot, v); }
__device__ __forceinline__ void slot_red(double *slot, cd v) {
    red_add(slot, v.re);
    red_add(slot + 1, v.im);
}

// Fused accumulation of row i's products in a sampling sweep (Eq. 1/C,
// P:173-176): z_i w_i^* into the diag slot and the pattern slot of (i, i);
// z_i w_j^* and z_j w_i^* for the lower neighbours j (final values, L1-hot
// from the gathers) into their pattern slots. Called by all 32 lanes of a
// converged warp (acc = false for lanes without a valid, active item).
template <typename S, int P, int V>
__device__ __forceinline__ void accumulate_row(const Sweep3Params<S> &p, const ZW<S> *zcol, int4 rec, S zi, S wi,
                                               bool acc, int lane, bool gleader, bool towner, double *sd,
                                               double *sp, bool want_diag, bool want_pat) {
    constexpr int E = ScalarTraits<S>::kDoubles;
    const int i = rec.x, beg = rec.y;
    if (want_diag || want_pat) {
        // z_i w_i^*: diag element i and pattern element (i, i)
        const S d = group_sum<P>(acc ? zwc_s(zi, wi) : zero_s<S>());
        if (acc && gleader) {
            if (want_diag) slot_red(sd + (int64_t)i * E, d);
            if (want_pat && rec.w >= 0) slot_red(sp + (int64_t)rec.w * E, d);
        }
    }
    if (!want_pat) return;
    // z_i w_j^* and z_j w_i^* for the lower neighbours j = col[beg + e], e < nlow
    const int nlow = acc ? rec.z >> 16 : 0;
    if constexpr (P == 1) {
        for (int e = 0; e < nlow; ++e) {
            const ZW<S> u = ld_zw(zcol + (int64_t)__ldg(p.ent_col + beg + e) * p.ld);
            const int2 pz = __ldg(p.ent_pz + beg + e);
            if (pz.x >= 0) slot_red(sp + (int64_t)pz.x * E, zwc_s(zi, u.w));
            if (pz.y >= 0) slot_red(sp + (int64_t)pz.y * E, zwc_s(u.z, wi));
        }
    } else {
        constexpr int VE = V / 2;  // entries per transpose-reduction
        const int nb = (__reduce_max_sync(0xffffffffu, nlow) + VE - 1) / VE;
        for (int b = 0; b < nb; ++b) {
            S v[V];
#pragma unroll
            for (int q = 0; q < VE; ++q) {
                const int e = b * VE + q;
                const int jc = __ldg(p.ent_col + beg + e);  // padded: always in bounds
                const bool ok = e < nlow;
                const ZW<S> u = ld_zw(zcol + (int64_t)(ok ? jc : 0) * p.ld);
                v[2 * q] = ok ? zwc_s(zi, u.w) : zero_s<S>();
                v[2 * q + 1] = ok ? zwc_s(u.z, wi) : zero_s<S>();
            }
            int held;
            const S x = transpose_sum<P, V>(v, lane, held);
            const int e = b * VE + (held >> 1);
            if (towner && e < nlow) {
                const int2 pz = __ldg(p.ent_pz + beg + e);
                const int slot = (held & 1) ? pz.y : pz.x;
                if (slot >= 0) slot_red(sp + (int64_t)slot * E, x);
            }
        }
    }
}

}  // namespace

template <typename S, int KU, int NT, int LGP>
__global__ void __launch_bounds__(NT, 1) sweep3_kernel(const Sweep3Params<S> p) {
    constexpr int E = ScalarTraits<S>::kDoubles;
    constexpr int P = 1 << LGP;        // lanes of one SE group inside this CTA (<= C)
    constexpr int V = P < 8 ? P : 8;   // products per transpose-reduction (pairs of one entry)
    const int tid = threadIdx.x;
    const int B = blockDim.x;  // a multiple of 32 and of C
    const int lane = tid & 31;
    const int wbase = tid - lane;
    const int lgC = p.lgC;
    const int C = 1 << lgC;
    const int c = tid & (C - 1);
    const int chain = (blockIdx.x << lgC) + c;
    const bool active = chain < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);
    const bool gleader = (c & (P - 1)) == 0;           // owner of a plain group sum
    const bool towner = (lane & ((P > V ? P / V : 1) - 1)) == 0;  // owner of a transposed value
    const int64_t grp = chain >> p.lgG;                // SE group of this chain = its accumulator slot
    ZW<S> *__restrict__ zcol = p.zw + chain;
    const bool want_diag = p.outputs & OUT_DIAG, want_pat = p.outputs & OUT_PATTERN;
    const bool want_tr = p.outputs & OUT_TRACE, want_full = p.outputs & OUT_FULL;
    double *const sd = p.slot_diag + grp * p.n * E;
    double *const sp = p.slot_pat + grp * p.pcount * E;
    S tr = zero_s<S>();

    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const int nph = sampling ? p.D + 1 : p.D;
        for (int ph = 0; ph < nph; ++ph) {
            // ---- row updates of level ph; warp-uniform trip count (shuffles below)
            const int r0 = __ldg(p.ph_row + ph);
            const int nu = (__ldg(p.ph_row + ph + 1) - r0) << lgC;
            for (int base = wbase; base < nu; base += B) {
                const int t = base + lane;
                const bool valid = t < nu;
                const int o = r0 + (t >> lgC);
                const int4 rec = valid ? __ldg(p.ord_rec + o) : make_int4(0, 0, 0, -1);
                const int i = rec.x, beg = rec.y, cnt = rec.z & 0xffff;
                S zi = zero_s<S>(), wi = zero_s<S>();
                if (valid) {
                    // noise first: its temporaries are dead before the gathers are in flight
                    double phi;
                    if (p.noise == 0) phi = gaussian(static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
                    else phi = p.noise == 2 ? 1.0 : 0.0;
                    S az = zero_s<S>(), aw = zero_s<S>();
                    row_sums<S, KU>(p, zcol, beg, cnt, az, aw);
                    const S dl = ldg_s(p.ord_dsg + 2 * o), sg = ldg_s(p.ord_dsg + 2 * o + 1);
                    zi = fma_s(neg_s(dl), az, scale_s(sg, phi));
                    wi = fma_s(neg_s(conj_s(dl)), aw, scale_s(conj_s(sg), phi));
                    zcol[(int64_t)i * p.ld] = ZW<S>{zi, wi};
                    if (want_full && sampling) {
                        const int64_t ts = s - p.snap_s0;
                        p.snap_x[(ts * p.n + i) * p.ld + chain] = zi;
                        p.snap_y[(ts * p.n + i) * p.ld + chain] = wi;
                    }
                }
                if (!sampling) continue;
                accumulate_row<S, P, V>(p, zcol, rec, zi, wi, valid && active, lane, gleader, towner, sd, sp,
                                        want_diag, want_pat);
            }
            if (sampling) {
                // ---- deferred trace items: conj(w_i) sum_j Q_ij z_j  (w^dagger Q z, reading R2);
                // per-thread register sums, no shuffles
                if (want_tr) {
                    const int q0 = __ldg(p.ph_tq + ph);
                    const int nq = (__ldg(p.ph_tq + ph + 1) - q0) << lgC;
                    for (int t = tid; t < nq; t += B) {
                        const int o = q0 + (t >> lgC);
                        const int i = __ldg(p.tq_row + o);
                        S qz = zero_s<S>();
                        for (int e = __ldg(p.tq_eptr + o); e < __ldg(p.tq_eptr + o + 1); ++e)
                            qz = add_s(qz, mul_s(ldg_s(p.tq_val + e),
                                                 ld_zw(zcol + (int64_t)__ldg(p.tq_col + e) * p.ld).z));
                        tr = add_s(tr, zwc_s(qz, ld_zw(zcol + (int64_t)i * p.ld).w));
                    }
                }
                // ---- deferred pattern pairs z_i w_j^*
                if (want_pat) {
                    const int q0 = __ldg(p.ph_pp + ph);
                    const int nq = (__ldg(p.ph_pp + ph + 1) - q0) << lgC;
                    for (int base = wbase; base < nq; base += B) {
                        const int t = base + lane;
                        const bool valid = t < nq;
                        const int o = q0 + (t >> lgC);
                        S x = zero_s<S>();
                        if (valid && active)
                            x = zwc_s(ld_zw(zcol + (int64_t)__ldg(p.pp_i + o) * p.ld).z,
                                      ld_zw(zcol + (int64_t)__ldg(p.pp_j + o) * p.ld).w);
                        x = group_sum<P>(x);
                        if (valid && active && gleader) slot_red(sp + (int64_t)__ldg(p.pp_slot + o) * E, x);
                    }
                }
            }
            __syncthreads();
        }
    }

    if (want_tr) {
        // per-chain trace: sum over the threads of each chain, then over the P chains of a group
        extern __shared__ __align__(16) unsigned char red_raw[];
        S *red = reinterpret_cast<S *>(red_raw);
        red[tid] = active ? tr : zero_s<S>();
        __syncthreads();
        if (wbase < C) {  // whole warps (C < 32: lanes >= C hold zeros and are not leaders)
            S v = zero_s<S>();
            if (tid < C)
                for (int h = tid; h < B; h += C) v = add_s(v, red[h]);
            v = group_sum<P>(v);
            if (tid < C && gleader && active) slot_red(p.slot_trace + grp * E, v);
        }
    }
}

// ---------------------------------------------------------------- v4: dataflow
//
// The same row update and accumulation, without per-level barriers. Every row
// j has a completion counter done[j] (shared memory, one byte, counted modulo
// 256) = the number of sweeps of this launch's chains that have updated it.
// Row i in sweep s may run once every lower neighbour j < i has done[j] >=
// s + 1 (its new value, Eq. 4/5 read order) and every upper neighbour has
// done[j] >= s: the upper neighbour has finished sweep s - 1, i.e. it has
// read z_i of sweep s - 1 (write-after-read) and holds the value row i must
// read. Neighbour counters differ by at most 2, so byte arithmetic is exact.
// Each warp takes groups of R = 32 / C rows (never spanning a level: rows of
// a group are independent) in increasing (sweep, level order); all
// dependencies point to earlier groups, so the earliest unfinished group can
// always run: no deadlock. A bounded wait (watchdog) reports instead of
// hanging if that reasoning were ever violated.
template <typename S, int KU, int NT, int LGP>
__global__ void __launch_bounds__(NT, 1) sweep4_kernel(const Sweep3Params<S> p) {
    constexpr int E = ScalarTraits<S>::kDoubles;
    constexpr int P = 1 << LGP;
    constexpr int V = P < 8 ? P : 8;
    extern __shared__ __align__(16) unsigned char done[];  // [n]
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    const int lane = tid & 31;
    const int lgC = p.lgC;  // C <= 32: the C lanes of a row are in one warp
    const int C = 1 << lgC;
    const int c = lane & (C - 1);
    const int chain = (blockIdx.x << lgC) + c;
    const bool active = chain < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);
    const bool gleader = (c & (P - 1)) == 0;
    const bool towner = (lane & ((P > V ? P / V : 1) - 1)) == 0;
    const int64_t grp = chain >> p.lgG;
    ZW<S> *__restrict__ zcol = p.zw + chain;
    const bool want_diag = p.outputs & OUT_DIAG, want_pat = p.outputs & OUT_PATTERN;
    const bool want_full = p.outputs & OUT_FULL;
    double *const sd = p.slot_diag + grp * p.n * E;
    double *const sp = p.slot_pat + grp * p.pcount * E;

    for (int j = tid; j < p.n; j += B) done[j] = static_cast<unsigned char>(p.s_begin);
    __syncthreads();

    const int R = 32 >> lgC;
    const int ngroups = p.nslots / R;
    const int64_t total = (int64_t)(p.s_end - p.s_begin) * ngroups;
    for (int64_t gi = tid >> 5; gi < total; gi += B >> 5) {
        const int s = p.s_begin + (int)(gi / ngroups);
        const int slot = (int)(gi % ngroups) * R + (lane >> lgC);
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const int4 rec = __ldg(p.slot_rec + slot);
        const bool valid = rec.x >= 0;
        const int i = rec.x, beg = rec.y, cnt = valid ? rec.z & 0xffff : 0;
        S zi = zero_s<S>(), wi = zero_s<S>();
        if (valid) {
            double phi;
            if (p.noise == 0) phi = gaussian(static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
            else phi = p.noise == 2 ? 1.0 : 0.0;
            // dependency wait (all C lanes of the row read the same counters: smem broadcast)
            const unsigned char lo = static_cast<unsigned char>(s + 1), hi = static_cast<unsigned char>(s);
            for (int e = 0; e < cnt; ++e) {
                const int j = __ldg(p.ent_col + beg + e);
                const unsigned char need = j < i ? lo : hi;
                const volatile unsigned char *f = done + j;
                if (static_cast<signed char>(*f - need) < 0) {
                    unsigned spins = 0;
                    while (static_cast<signed char>(*f - need) < 0 && !*reinterpret_cast<volatile unsigned *>(p.err)) {
                        __nanosleep(32);
                        if (++spins > (1u << 26)) {  // ~seconds: report, do not hang
                            atomicOr(p.err, 1u);
                            break;
                        }
                    }
                }
            }
            __threadfence_block();  // acquire: gathers after the counters
            S az = zero_s<S>(), aw = zero_s<S>();
            row_sums<S, KU>(p, zcol, beg, cnt, az, aw);
            const S dl = ldg_s(p.slot_dsg + 2 * slot), sg = ldg_s(p.slot_dsg + 2 * slot + 1);
            zi = fma_s(neg_s(dl), az, scale_s(sg, phi));
            wi = fma_s(neg_s(conj_s(dl)), aw, scale_s(conj_s(sg), phi));
            zcol[(int64_t)i * p.ld] = ZW<S>{zi, wi};
            if (want_full && sampling) {
                const int64_t ts = s - p.snap_s0;
                p.snap_x[(ts * p.n + i) * p.ld + chain] = zi;
                p.snap_y[(ts * p.n + i) * p.ld + chain] = wi;
            }
        }
        __syncwarp();  // the row's C stores are ordered before its counter update
        if (valid && c == 0) {
            __threadfence_block();  // release
            *reinterpret_cast<volatile unsigned char *>(done + i) = static_cast<unsigned char>(s + 1);
        }
        if (sampling)
            accumulate_row<S, P, V>(p, zcol, rec, zi, wi, valid && active, lane, gleader, towner, sd, sp, want_diag,
                                    want_pat);
    }
}

namespace {

template <typename S, int LGP>
cudaError_t launch3(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    // gathers in flight per row chunk: 64 registers at 1024 threads, 85 at 768, 128 at 512
    // (the entry arrays are padded by 8 entries: KU <= 8)
    constexpr int KS = ScalarTraits<S>::kDoubles == 1 ? 4 : 2;
    const int C = 1 << p.lgC;
    const int blocks = (p.chains + C - 1) / C;
    const size_t smem = (p.outputs & OUT_TRACE) ? (size_t)threads * sizeof(S) : 0;
    if (threads <= 512) sweep3_kernel<S, 2 * KS, 512, LGP><<<blocks, threads, smem, st>>>(p);
    else if (threads <= 768) sweep3_kernel<S, KS, 768, LGP><<<blocks, threads, smem, st>>>(p);
    else sweep3_kernel<S, KS, 1024, LGP><<<blocks, threads, smem, st>>>(p);
    return cudaGetLastError();
}

}  // namespace

template <typename S, int LGP>
cudaError_t launch4(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    constexpr int KS = ScalarTraits<S>::kDoubles == 1 ? 4 : 2;
    const int C = 1 << p.lgC;
    const int blocks = (p.chains + C - 1) / C;
    const size_t smem = ((size_t)p.n + 15) / 16 * 16;
    cudaError_t e;
    if (threads <= 512) {
        auto k = sweep4_kernel<S, 2 * KS, 512, LGP>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) k<<<blocks, threads, smem, st>>>(p);
    } else if (threads <= 768) {
        auto k = sweep4_kernel<S, KS, 768, LGP>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) k<<<blocks, threads, smem, st>>>(p);
    } else {
        auto k = sweep4_kernel<S, KS, 1024, LGP>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) k<<<blocks, threads, smem, st>>>(p);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
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
template cudaError_t launch_sweep4<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep4<cd>(const Sweep3Params<cd> &, int, cudaStream_t);
template cudaError_t launch_sweep3<cd>(const Sweep3Params<cd> &, int, cudaStream_t);

}  // namespace mcinv
