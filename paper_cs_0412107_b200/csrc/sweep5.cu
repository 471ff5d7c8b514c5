// sweep5.cu -- K1/K2 (v5): the dataflow sweep kernel of v4 (sweep3.cu) with
// the plan data of every warp group staged into shared memory by TMA bulk
// copies. Same row update (Eq. 4/5), same accumulation
// (Eq. 1/C) and the same bit-identical operand order as the
// sequential row loop; see DESIGN.md "K1 sweep5_kernel".
#include <cstdlib>

#include "sweep_common.cuh"

namespace mcinv {
// ---------------------------------------------------------------- v5: v4 + TMA-staged plan
//
// The dataflow kernel of v4 with the plan data of every warp group (row
// records, delta/sigma, entry columns, coefficient pairs, pattern slots)
// packed by the host into one contiguous block and staged into a per-warp,
// double-buffered shared-memory slot by a TMA bulk copy (cp.async.bulk +
// mbarrier complete_tx) one group ahead: the dependency checks, the gathers'
// addresses and coefficients and the accumulation's partners and slots then
// read shared memory, and the unified L1 is left to the state lines.
namespace {

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
    const int nlow = acc ? static_cast<int>(static_cast<unsigned>(rec.z) >> 16) : 0;
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
// GAUSS: the run's noise is the Gaussian one (the default; compile-time: +1.4% config 2, +2.5%
// config 3 over the run-time switch between the noise modes)
template <typename S, int KU, int NT, int LGC, int LGP, bool BITS, bool GAUSS>
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
    // (a compile-time flag here measured 2% slower: code generation in this register-capped
    // kernel is fragile; removing unused runtime branches -- prefetch variants, optional
    // reconvergence, sleep in the polls -- measured +5% on config 2)
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
    bool dv = false;  // divergence seen (reading R12: every stored value is a sweep-end value)
    const bool want_tr = p.outputs & OUT_TRACE;
    S tr = zero_s<S>(), trs = zero_s<S>();  // the chain's trace over the launch / over the current sweep
    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const unsigned char need = static_cast<unsigned char>(s + 1);
        for (int g = w; g < ngroups; g += W, ++item) {
            const bool odd = item & 1;
            unsigned char *cur = odd ? buf1 : buf0;
            // stage the next group (this warp's next item, possibly in the next sweep) into the
            // other slot: the previous item's reads of it are complete (its closing __syncwarp)
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
            if (rec.x <= -2) {
                // a trace item of row -2 - rec.x (scheduled after rows i and j of its Q row, whose
                // sweep-s values then hold until the sweep barrier): entries [i, Q cols], waited
                // for, then conj(w_i) sum_j Q_ij z_j (Eq. tr, reading R2). Sampling sweeps only.
                if (sampling) {
                    const int tc = rec.z & 0xffff;
                    for (int e = 0; e < tc; ++e) {
                        const int j = col[e];
                        auto ready = [&]() -> bool {
                            if constexpr (BITS)
                                return ((reinterpret_cast<volatile unsigned *>(dbits)[j >> 5] >> (j & 31)) & 1u) ==
                                       (need & 1u);
                            else
                                return reinterpret_cast<volatile unsigned char *>(done)[j] == need;
                        };
                        wait_ready(ready, p.err, 0);
                    }
                    __threadfence_block();  // acquire
                    // w_i and the first gathers of z_j all in flight before the products
                    constexpr int TU = 4;
                    const S wt = ld_zw(zrow(zcol, col[0], zst)).w;
                    S zj[TU];
#pragma unroll
                    for (int q = 0; q < TU; ++q) zj[q] = 1 + q < tc ? ld_zw(zrow(zcol, col[1 + q], zst)).z : zero_s<S>();
                    S qz = zero_s<S>();
#pragma unroll
                    for (int q = 0; q < TU; ++q)
                        if (1 + q < tc) qz = add_s(qz, mul_s(ab[1 + q].z, zj[q]));
                    for (int e = 1 + TU; e < tc; ++e) qz = add_s(qz, mul_s(ab[e].z, ld_zw(zrow(zcol, col[e], zst)).z));
                    trs = add_s(trs, zwc_s(qz, wt));
                }
                // (then on through the warp's collective steps as an invalid row: no update,
                // no publication, zero products)
            }
            if (valid) {
                const int nlow = static_cast<int>(static_cast<unsigned>(rec.z) >> 16);
                // upper neighbours hold their sweep s-1 values until this row publishes: start
                // their lines on the way before the noise (its ALU time covers the latency)
                if (p.prefetch) {  // all neighbours into L2 (the coherence point: safe for lower ones)
                    for (int e0 = 0; e0 < cnt; e0 += KU)  // KU-padded entry lists: no predicate
#pragma unroll
                        for (int q = 0; q < KU; ++q) prefetch_l2(zrow(zcol, col[e0 + q], zst));
                }
                if constexpr (GAUSS)
                    phi = gaussian(static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
                else
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
                    wait_ready(ready, p.err, 0);  // busy poll (measured best; MCINV_SPIN_NS is v4's)
                }
            }
            if (valid) {
                __threadfence_block();  // acquire (the polls are relaxed loads; acquire loads measured ±0.5%)
                S az = zero_s<S>(), aw = zero_s<S>();
                row_sums_blk<S, KU>(p, zcol, col, ab, cnt, az, aw);
                const S dl = dsg[0], sg = dsg[1];
                zi = fma_s(neg_s(dl), az, scale_s(sg, phi));
                wi = fma_s(neg_s(conj_s(dl)), aw, scale_s(conj_s(sg), phi));
                *zrow(zcol, i, zst) = ZW<S>{zi, wi};
                dv = dv | bad_s(zi) | bad_s(wi);
                if (want_full && sampling) {
                    const int64_t ts = s - p.snap_s0;
                    p.snap_x[(ts * p.n + i) * p.ld + chain] = zi;
                    p.snap_y[(ts * p.n + i) * p.ld + chain] = wi;
                }
            }
            __syncwarp();  // the row's stores are ordered before its counter update
            if (valid && c == 0) {
                if constexpr (BITS) {
                    __threadfence_block();  // release
                    atomicXor(dbits + (i >> 5), 1u << (i & 31));
                } else {  // a release store instead of fence + store (+0.3%, config 3 +1.7%)
                    const unsigned short v = need;
                    asm volatile("st.release.cta.shared::cta.u8 [%0], %1;" ::"r"(smem_addr(done + i)), "h"(v)
                                 : "memory");
                }
            }
            if (sampling)
                accumulate_blk<S, P, V>(p, zcol, rec, col, pz, zi, wi, valid && active, lane, gleader, towner, sd,
                                        sp, want_diag, want_pat);
            // reconverge before the next item: lanes that skipped a divergent step of the
            // accumulation (leaders' reductions) otherwise start it as a separate sub-warp and
            // the split persists (diag-only config 2: 1.57e10 without, 2.79e10 with); it also
            // orders every lane's reads of this item's block before the next item's TMA into it
            __syncwarp();
        }
        if (want_tr && sampling) {  // Geyer's series: this sweep's realized trace of the warp's chains
            if (p.series) {
                const S v = group_sum<32>(active ? trs : zero_s<S>());
                if (lane == 0) slot_red(p.series + (int64_t)(p.series_base + s - p.burn_in) * E, v);
            }
            tr = add_s(tr, trs);
            trs = zero_s<S>();
        }
        __syncthreads();  // sweep boundary: all reads of sweep s values are done
    }
    if (dv && active) atomicAdd(p.bad, 1.0);
    if (want_tr) {
        // per-chain trace: sum over the threads of each chain (shared memory, the block area is
        // free after the last barrier), then over the P chains of a group, one red per group
        S *red = reinterpret_cast<S *>(sm5);
        red[tid] = active ? tr : zero_s<S>();
        __syncthreads();
        if (w == 0) {  // C <= 32: the chains' sums in the lanes c < C of warp 0
            S v = zero_s<S>();
            if (lane < C)
                for (int h = lane; h < B; h += C) v = add_s(v, red[h]);
            v = group_sum<P>(v);
            if (lane < C && gleader && active) slot_red(p.slot_trace + grp * E, v);
        }
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
    constexpr int NT = kReal ? 1024 : 768, KU = kReal ? MCINV_V5_KUR : MCINV_V5_KUC;
    if (threads > NT) return cudaErrorInvalidConfiguration;
    const int blocks = (p.chains + (1 << LGC) - 1) >> LGC;
    size_t smem = sweep5_smem(p.n, threads, p.maxb);
    if ((p.outputs & OUT_TRACE) && smem < (size_t)threads * sizeof(S)) smem = (size_t)threads * sizeof(S);
    // the Gaussian-only variant for byte counters (the common case); bit counters keep the switch
    auto k = (!BITS && p.noise == 0) ? sweep5_kernel<S, KU, NT, LGC, LGP, BITS, !BITS>
                                     : sweep5_kernel<S, KU, NT, LGC, LGP, BITS, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // the smallest shared-memory carveout that holds the CTA: the rest of the unified L1
    // caches state lines
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

}  // namespace mcinv
