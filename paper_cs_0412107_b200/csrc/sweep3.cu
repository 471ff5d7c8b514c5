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
#include <type_traits>

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

// &zcol[j * ld] as one IMAD.WIDE.U32 (32 x 32 -> 64-bit product plus the base) instead of
// a 64-bit multiply and shift: j < 2^31 and the row stride in bytes (ld * sizeof) < 2^32
template <typename T>
__device__ __forceinline__ T *zrow(T *zcol, int j, uint32_t stride) {
    using C = typename std::conditional<std::is_const<T>::value, const char, char>::type;
    return reinterpret_cast<T *>(reinterpret_cast<C *>(zcol) + static_cast<uint64_t>(static_cast<uint32_t>(j)) * stride);
}

__device__ __forceinline__ void prefetch_l1(const void *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
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

// K consecutive (z, w) state elements of one row (K chains of a thread) in
// 256-bit accesses where they fill one (LDG.E.ENL2.256 on sm_100a).
template <typename S, int K>
struct ZWK {
    ZW<S> v[K];
};
__device__ __forceinline__ void ld256(const void *p, double &a, double &b, double &c, double &d) {
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
}
__device__ __forceinline__ void st256(void *p, double a, double b, double c, double d) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
template <typename S, int K>
__device__ __forceinline__ ZWK<S, K> ld_zwk(const ZW<S> *p) {
    ZWK<S, K> r;
    if constexpr (ScalarTraits<S>::kDoubles == 1 && K == 1) {
        r.v[0] = *p;
    } else if constexpr (ScalarTraits<S>::kDoubles == 1) {
#pragma unroll
        for (int q = 0; q < K; q += 2) ld256(p + q, r.v[q].z, r.v[q].w, r.v[q + 1].z, r.v[q + 1].w);
    } else {
#pragma unroll
        for (int q = 0; q < K; ++q) ld256(p + q, r.v[q].z.re, r.v[q].z.im, r.v[q].w.re, r.v[q].w.im);
    }
    return r;
}
template <typename S, int K>
__device__ __forceinline__ void st_zwk(ZW<S> *p, const ZWK<S, K> &r) {
    if constexpr (ScalarTraits<S>::kDoubles == 1 && K == 1) {
        *p = r.v[0];
    } else if constexpr (ScalarTraits<S>::kDoubles == 1) {
#pragma unroll
        for (int q = 0; q < K; q += 2) st256(p + q, r.v[q].z, r.v[q].w, r.v[q + 1].z, r.v[q + 1].w);
    } else {
#pragma unroll
        for (int q = 0; q < K; ++q) st256(p + q, r.v[q].z.re, r.v[q].z.im, r.v[q].w.re, r.v[q].w.im);
    }
}

// fma chains of Eq. (4)/(5) over the cnt entries at beg for the K chains of
// this thread, KU gathers in flight. Branch-free: the entry arrays are padded
// by 8 entries, so every load is unconditional; slots past the row's end
// gather row 0 of these chains (an L1-hot dummy) and their fma is predicated
// off, so the sums are exactly the serial ones.
template <typename S, int KU, int K>
__device__ __forceinline__ void row_sums(const Sweep3Params<S> &p, const ZW<S> *zcol, int beg, int cnt,
                                         S (&az)[K], S (&aw)[K]) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    for (int e0 = 0; e0 < cnt; e0 += KU) {
        int j[KU];
        ZWK<S, K> v[KU];
        ZW<S> ab[KU];
#pragma unroll
        for (int q = 0; q < KU; ++q) j[q] = __ldg(p.ent_col + beg + e0 + q);
#pragma unroll
        for (int q = 0; q < KU; ++q) {
            v[q] = ld_zwk<S, K>(zrow(zcol, (e0 + q < cnt ? j[q] : 0), zst));
            ab[q] = ldg_ab(reinterpret_cast<const ZW<S> *>(p.ent_ab) + beg + e0 + q);
        }
#pragma unroll
        for (int q = 0; q < KU; ++q)
            if (e0 + q < cnt) {
#pragma unroll
                for (int h = 0; h < K; ++h) {
                    az[h] = fma_s(ab[q].z, v[q].v[h].z, az[h]);
                    aw[h] = fma_s(ab[q].w, v[q].v[h].w, aw[h]);
                }
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
// from the gathers) into their pattern slots. The K chains of the thread are
// summed in registers (they belong to one SE group), then the P lanes of the
// group. Called by all 32 lanes of a converged warp; acc[h] = false for
// chains without a valid, active item.
template <typename S, int P, int V, int K>
__device__ __forceinline__ void accumulate_row(const Sweep3Params<S> &p, const ZW<S> *zcol, int4 rec, const S (&zi)[K],
                                               const S (&wi)[K], const bool (&acc)[K], int lane, bool gleader,
                                               bool towner, double *sd, double *sp, bool want_diag, bool want_pat) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    constexpr int E = ScalarTraits<S>::kDoubles;
    const int i = rec.x, beg = rec.y;
    bool any = false;
#pragma unroll
    for (int h = 0; h < K; ++h) any = any || acc[h];
    if (want_diag || want_pat) {
        // z_i w_i^*: diag element i and pattern element (i, i)
        S d = zero_s<S>();
#pragma unroll
        for (int h = 0; h < K; ++h)
            if (acc[h]) d = add_s(d, zwc_s(zi[h], wi[h]));
        d = group_sum<P>(d);
        if (any && gleader) {
            if (want_diag) slot_red(sd + (int64_t)i * E, d);
            if (want_pat && rec.w >= 0) slot_red(sp + (int64_t)rec.w * E, d);
        }
    }
    if (!want_pat) return;
    // z_i w_j^* and z_j w_i^* for the lower neighbours j = col[beg + e], e < nlow
    const int nlow = any ? rec.z >> 16 : 0;
    if constexpr (P == 1) {
        for (int e = 0; e < nlow; ++e) {
            const ZWK<S, K> u = ld_zwk<S, K>(zrow(zcol, __ldg(p.ent_col + beg + e), zst));
            S x = zero_s<S>(), y = zero_s<S>();
#pragma unroll
            for (int h = 0; h < K; ++h)
                if (acc[h]) {
                    x = add_s(x, zwc_s(zi[h], u.v[h].w));
                    y = add_s(y, zwc_s(u.v[h].z, wi[h]));
                }
            const int2 pz = __ldg(p.ent_pz + beg + e);
            if (pz.x >= 0) slot_red(sp + (int64_t)pz.x * E, x);
            if (pz.y >= 0) slot_red(sp + (int64_t)pz.y * E, y);
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
                const ZWK<S, K> u = ld_zwk<S, K>(zrow(zcol, (ok ? jc : 0), zst));
                S x = zero_s<S>(), y = zero_s<S>();
#pragma unroll
                for (int h = 0; h < K; ++h)
                    if (acc[h]) {
                        x = add_s(x, zwc_s(zi[h], u.v[h].w));
                        y = add_s(y, zwc_s(u.v[h].z, wi[h]));
                    }
                v[2 * q] = ok ? x : zero_s<S>();
                v[2 * q + 1] = ok ? y : zero_s<S>();
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

template <typename S, int KU, int NT, int LGP, int K>
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
    S tr = zero_s<S>();  // K == 1 only (trace runs use K = 1)

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
#pragma unroll
                    for (int h = 0; h < K; ++h) {
                        phi[h] = noise_phi(p.noise, static_cast<uint32_t>(i), k,
                                           p.chain0 + static_cast<uint32_t>(chain + h), p.key0, p.key1);
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
                            tr = add_s(tr, zwc_s(qz, ld_zw(zrow(zcol, i, zst)).w));
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
    }

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
// Dataflow wait: poll a shared-memory counter until ready(). The global abort flag
// (watchdog: another warp gave up) is read only every 256 polls: reading it on every poll
// put a global-load latency between a counter's publication and its waiter seeing it
// (ncu: ~19% of v5's stall samples sat on that load). A wait of ~seconds sets the flag.
template <typename F>
__device__ __forceinline__ void wait_ready(F ready, unsigned *err, int spin_ns) {
    if (ready()) return;
    for (unsigned spins = 1;; ++spins) {
        if (spin_ns > 0) {
            __nanosleep(spin_ns);
            if (ready()) return;
        } else {  // busy poll: 8 polls per round (a load, a compare and a branch each)
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (ready()) return;
        }
        if ((spins & 63u) == 0) {
            if (*reinterpret_cast<volatile unsigned *>(err)) return;
            if (spins > (1u << 26)) {
                atomicOr(err, 1u);
                return;
            }
        }
    }
}

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
                const int nlow = rec.z >> 16;
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
        }
        __syncthreads();  // sweep boundary: all reads of sweep s values are done
    }
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

// ---------------------------------------------------------------- v5: v4 + TMA-staged plan
constexpr int kByteCounters = 160000;  // larger n: one completion bit per row
//
// The dataflow kernel of v4 with the plan data of every warp group (row
// records, delta/sigma, entry columns, coefficient pairs, pattern slots)
// packed by the host into one contiguous block and staged into a per-warp,
// double-buffered shared-memory slot by a TMA bulk copy (cp.async.bulk +
// mbarrier complete_tx) one group ahead: the dependency checks, the gathers'
// addresses and coefficients and the accumulation's partners and slots then
// read shared memory, and the unified L1 is left to the state lines.
namespace {

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void tma_block(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our generic reads of this slot precede
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Eq. (4)/(5) fma chains from a staged block (see row_sums): the host padded the row's
// entries to a multiple of KU with zero coefficients on a valid column, so the unrolled
// chain runs unpredicated
template <typename S, int KU>
__device__ __forceinline__ void row_sums_blk(const Sweep3Params<S> &p, const ZW<S> *zcol, const int *col,
                                             const ZW<S> *ab, int cnt, S &az, S &aw) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    for (int e0 = 0; e0 < cnt; e0 += KU) {
        int j[KU];
        ZW<S> v[KU], c[KU];
#pragma unroll
        for (int q = 0; q < KU; ++q) j[q] = col[e0 + q];
#pragma unroll
        for (int q = 0; q < KU; ++q) {
            v[q] = ld_zw(zrow(zcol, j[q], zst));
            c[q] = ab[e0 + q];
        }
#pragma unroll
        for (int q = 0; q < KU; ++q) {
            az = fma_s(c[q].z, v[q].z, az);
            aw = fma_s(c[q].w, v[q].w, aw);
        }
    }
}

// accumulation as accumulate_row (K = 1), partners' columns and slots from the block
template <typename S, int P, int V>
__device__ __forceinline__ void accumulate_blk(const Sweep3Params<S> &p, const ZW<S> *zcol, int4 rec, const int *col,
                                               const int2 *pz, S zi, S wi, bool acc, int lane, bool gleader,
                                               bool towner, double *sd, double *sp, bool want_diag, bool want_pat) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    constexpr int E = ScalarTraits<S>::kDoubles;
    const int i = rec.x;
    if (want_diag || want_pat) {
        const S d = group_sum<P>(acc ? zwc_s(zi, wi) : zero_s<S>());
        if (acc && gleader) {
            if (want_diag) slot_red(sd + (int64_t)i * E, d);
            if (want_pat && rec.w >= 0) slot_red(sp + (int64_t)rec.w * E, d);
        }
    }
    if (!want_pat) return;
    const int nlow = acc ? rec.z >> 16 : 0;
    if constexpr (P == 1) {
        for (int e = 0; e < nlow; ++e) {
            const ZW<S> u = ld_zw(zrow(zcol, col[e], zst));
            const int2 z2 = pz[e];
            if (z2.x >= 0) slot_red(sp + (int64_t)z2.x * E, zwc_s(zi, u.w));
            if (z2.y >= 0) slot_red(sp + (int64_t)z2.y * E, zwc_s(u.z, wi));
        }
    } else {
        constexpr int VE = V / 2;
        const int nb = (__reduce_max_sync(0xffffffffu, nlow) + VE - 1) / VE;
        for (int b = 0; b < nb; ++b) {
            S v[V];
#pragma unroll
            for (int q = 0; q < VE; ++q) {
                const int e = b * VE + q;
                const bool ok = e < nlow;
                const ZW<S> u = ld_zw(zrow(zcol, (ok ? col[e] : 0), zst));
                v[2 * q] = ok ? zwc_s(zi, u.w) : zero_s<S>();
                v[2 * q + 1] = ok ? zwc_s(u.z, wi) : zero_s<S>();
            }
            int held;
            const S x = transpose_sum<P, V>(v, lane, held);
            const int e = b * VE + (held >> 1);
            if (towner && e < nlow) {
                const int2 z2 = pz[e];
                const int slot = (held & 1) ? z2.y : z2.x;
                if (slot >= 0) slot_red(sp + (int64_t)slot * E, x);
            }
        }
    }
}

}  // namespace

// BITS: one completion bit per row instead of a byte (n up to ~1.8M rows in shared memory):
// with the sweep barrier a row's counter only has to tell "updated in this sweep" from
// "in the previous one", i.e. its parity; publishing toggles the bit (atomicXor).
template <typename S, int KU, int NT, int LGC, int LGP, bool BITS>
__global__ void __launch_bounds__(NT, 1) sweep5_kernel(const Sweep3Params<S> p) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<S>));
    constexpr int E = ScalarTraits<S>::kDoubles;
    constexpr int P = 1 << LGP;
    constexpr int V = P < 8 ? P : 8;
    extern __shared__ __align__(128) unsigned char sm5[];
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    const int W = B >> 5;
    const int w = tid >> 5;
    const int lane = tid & 31;
    constexpr int lgC = LGC;  // C <= 32: a row's lanes are in one warp (compile-time: R, sub, c)
    constexpr int C = 1 << lgC;
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
    // shared memory: [W][2] mbarriers | [W][2][maxb] block slots | done[n]
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm5);
    unsigned char *blk = sm5 + 16 * W;
    unsigned char *done = blk + (size_t)2 * W * p.maxb;
    unsigned *dbits = reinterpret_cast<unsigned *>(done);
    const uint32_t bar0 = smem_addr(bars + 2 * w), bar1 = bar0 + 8;
    unsigned char *buf0 = blk + (size_t)2 * w * p.maxb, *buf1 = buf0 + p.maxb;

    if constexpr (BITS) {
        const unsigned fill = (p.s_begin & 1) ? 0xffffffffu : 0u;
        for (int j = tid; j < (p.n + 31) / 32; j += B) dbits[j] = fill;
    } else {
        for (int j = tid; j < p.n; j += B) done[j] = static_cast<unsigned char>(p.s_begin);
    }
    if (lane == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    constexpr int R = 32 >> lgC;
    const int ngroups = p.nslots / R;
    const int sub = lane >> lgC;
    auto issue = [&](int g, unsigned char *dst, uint32_t bar) {
        const int64_t off = __ldg(p.gofs + g);
        const uint32_t bytes = static_cast<uint32_t>(__ldg(p.gofs + g + 1) - off);
        tma_block(smem_addr(dst), p.blob + off, bytes, bar);
    };
    if (lane == 0 && w < ngroups) issue(w, buf0, bar0);
    uint32_t ph0 = 0, ph1 = 0;
    int item = 0;
    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const unsigned char need = static_cast<unsigned char>(s + 1);
        for (int g = w; g < ngroups; g += W, ++item) {
            const bool odd = item & 1;
            unsigned char *cur = odd ? buf1 : buf0;
            // stage the next group (this warp's next item, possibly in the next sweep) into the
            // other slot: the previous item's reads of it are complete (__syncwarp)
            __syncwarp();
            const int gn = g + W < ngroups ? g + W : w;
            const bool has_next = g + W < ngroups || s + 1 < p.s_end;
            if (lane == 0 && has_next) issue(gn, odd ? buf0 : buf1, odd ? bar0 : bar1);
            if (odd) {
                mbar_wait(bar1, ph1);
                ph1 ^= 1;
            } else {
                mbar_wait(bar0, ph0);
                ph0 ^= 1;
            }
            const int4 head = reinterpret_cast<const int4 *>(cur)[0];
            const int4 rec = reinterpret_cast<const int4 *>(cur)[1 + sub];
            const int *col = reinterpret_cast<const int *>(cur + 16 + 16 * R + 2 * sizeof(S) * R) + rec.y;
            const ZW<S> *ab = reinterpret_cast<const ZW<S> *>(cur + head.z) + rec.y;
            const int2 *pz = reinterpret_cast<const int2 *>(cur + head.w) + rec.y;
            const S *dsg = reinterpret_cast<const S *>(cur + 16 + 16 * R) + 2 * sub;
            const bool valid = rec.x >= 0;
            const int i = rec.x, cnt = valid ? rec.z & 0xffff : 0;
            S zi = zero_s<S>(), wi = zero_s<S>();
            double phi = 0.0;
            if (valid) {
                const int nlow = rec.z >> 16;
                // upper neighbours hold their sweep s-1 values until this row publishes: start
                // their lines on the way before the noise (its ALU time covers the latency)
                if (p.prefetch == 3) {  // all neighbours into L2 (the coherence point: safe for lower ones)
                    for (int e0 = 0; e0 < cnt; e0 += KU)  // KU-padded entry lists: no predicate
#pragma unroll
                        for (int q = 0; q < KU; ++q) prefetch_l2(zrow(zcol, col[e0 + q], zst));
                } else if (p.prefetch == 1) {
                    for (int e = nlow; e < cnt; ++e) prefetch_l1(zrow(zcol, col[e], zst));
                } else if (p.prefetch == 2) {
                    for (int e = nlow; e < cnt; ++e) prefetch_l2(zrow(zcol, col[e], zst));
                }
                phi = noise_phi(p.noise, static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
                for (int e = 0; e < nlow; ++e) {
                    const int j = col[e];
                    auto ready = [&]() -> bool {
                        if constexpr (BITS)
                            return ((reinterpret_cast<volatile unsigned *>(dbits)[j >> 5] >> (j & 31)) & 1u) ==
                                   (need & 1u);
                        else
                            return reinterpret_cast<volatile unsigned char *>(done)[j] == need;
                    };
                    wait_ready(ready, p.err, p.spin_ns);
                }
            }
            // rows whose dependencies were ready left the wait early; reconverge so that the
            // gathers and the fma chains of the warp's R rows issue as one instruction stream
            if (p.reconv & 2) __syncwarp();
            if (valid) {
                __threadfence_block();
                S az = zero_s<S>(), aw = zero_s<S>();
                row_sums_blk<S, KU>(p, zcol, col, ab, cnt, az, aw);
                const S dl = dsg[0], sg = dsg[1];
                zi = fma_s(neg_s(dl), az, scale_s(sg, phi));
                wi = fma_s(neg_s(conj_s(dl)), aw, scale_s(conj_s(sg), phi));
                *zrow(zcol, i, zst) = ZW<S>{zi, wi};
                if (want_full && sampling) {
                    const int64_t ts = s - p.snap_s0;
                    p.snap_x[(ts * p.n + i) * p.ld + chain] = zi;
                    p.snap_y[(ts * p.n + i) * p.ld + chain] = wi;
                }
            }
            __syncwarp();  // the row's stores are ordered before its counter update
            if (valid && c == 0) {
                __threadfence_block();  // release
                if constexpr (BITS) atomicXor(dbits + (i >> 5), 1u << (i & 31));
                else *reinterpret_cast<volatile unsigned char *>(done + i) = need;
            }
            if (sampling)
                accumulate_blk<S, P, V>(p, zcol, rec, col, pz, zi, wi, valid && active, lane, gleader, towner, sd,
                                        sp, want_diag, want_pat);
            // reconverge before the next item: lanes that skipped a divergent step of the
            // accumulation (leaders' reductions) otherwise start it as a separate sub-warp and
            // the split persists (diag-only config 2: 1.57e10 without, 2.79e10 with)
            if (p.reconv & 1) __syncwarp();
        }
        __syncthreads();  // sweep boundary: all reads of sweep s values are done
    }
}

size_t sweep5_smem(int n, int threads, int maxb) {
    const size_t W = (size_t)threads / 32;
    const size_t counters = n > kByteCounters ? ((size_t)n + 127) / 128 * 16 : ((size_t)n + 15) / 16 * 16;
    return 16 * W + 2 * W * (size_t)maxb + counters;
}

namespace {

// one thread count per scalar type (1024 real, 768 complex: the register budget of one
// CTA per SM); C and the group lanes P are template parameters (compile-time R, lane maps)
template <typename S, int LGC, int LGP, bool BITS>
cudaError_t launch5b(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    constexpr bool kReal = ScalarTraits<S>::kDoubles == 1;
    constexpr int NT = kReal ? 1024 : 768, KU = kReal ? 4 : 2;
    if (threads > NT) return cudaErrorInvalidConfiguration;
    const int blocks = (p.chains + (1 << LGC) - 1) >> LGC;
    const size_t smem = sweep5_smem(p.n, threads, p.maxb);
    auto k = sweep5_kernel<S, KU, NT, LGC, LGP, BITS>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // the smallest shared-memory carveout that holds the CTA: the rest of the unified L1
    // caches state lines (left to the driver, the carveout varied with the block size:
    // diag-only config 2 ran 1.6e10 against 2.3e10 with pattern blocks)
    int carve = (int)((smem + 8192) * 100 / (228 * 1024)) + 1;
    if (const char *ev = std::getenv("MCINV_CARVE")) carve = std::atoi(ev);
    if (carve >= 0) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve > 100 ? 100 : carve);
        if (e != cudaSuccess) return e;
    }
    k<<<blocks, threads, smem, st>>>(p);
    return cudaGetLastError();
}

template <typename S, int LGC, int LGP>
cudaError_t launch5(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    if constexpr (LGP > LGC) {
        return cudaErrorInvalidValue;
    } else {
        return p.n > kByteCounters ? launch5b<S, LGC, LGP, true>(p, threads, st)
                                   : launch5b<S, LGC, LGP, false>(p, threads, st);
    }
}

template <typename S, int LGC>
cudaError_t launch5c(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    switch (p.lgP) {
        case 0: return launch5<S, LGC, 0>(p, threads, st);
        case 1: return launch5<S, LGC, 1>(p, threads, st);
        case 2: return launch5<S, LGC, 2>(p, threads, st);
        case 3: return launch5<S, LGC, 3>(p, threads, st);
        case 4: return launch5<S, LGC, 4>(p, threads, st);
        case 5: return launch5<S, LGC, 5>(p, threads, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

template <typename S>
cudaError_t launch_sweep5(const Sweep3Params<S> &p, int threads, cudaStream_t st) {
    switch (p.lgC) {
        case 0: return launch5c<S, 0>(p, threads, st);
        case 1: return launch5c<S, 1>(p, threads, st);
        case 2: return launch5c<S, 2>(p, threads, st);
        case 3: return launch5c<S, 3>(p, threads, st);
        case 4: return launch5c<S, 4>(p, threads, st);
        case 5: return launch5c<S, 5>(p, threads, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_sweep5<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep5<cd>(const Sweep3Params<cd> &, int, cudaStream_t);
template cudaError_t launch_sweep3<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep4<double>(const Sweep3Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep4<cd>(const Sweep3Params<cd> &, int, cudaStream_t);
template cudaError_t launch_sweep3<cd>(const Sweep3Params<cd> &, int, cudaStream_t);

}  // namespace mcinv
