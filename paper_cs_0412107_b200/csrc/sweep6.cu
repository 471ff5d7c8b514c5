// sweep6.cu -- K1/K2 (v6): the v5 dataflow kernel (sweep5.cu) with TWO chains per
// thread, for real C. Same row update (Eq. 4/5), same fused
// accumulation (Eq. 1/C), same bit-identical operand order as the
// sequential row loop; see DESIGN.md "K1 sweep6_kernel".
//
// A thread holds the adjacent chains 2m, 2m + 1 of one row: they are the two
// outputs of one Box-Muller pair (reading R4), so the noise -- Philox, ln, sqrt and
// the range reduction, the largest single cost of a site update -- is evaluated
// once per two sites; every gather is one 32-B load of both chains' (z, w); the
// per-row costs (dependency polls, plan reads, prefetches, the block staging)
// are paid once per two sites; and the accumulation pre-sums the two chains
// before the lane-group reduction. A warp item covers R = 64 / C rows of the CTA's
// C chains (C / 2 lanes per row).
#include <cstdio>
#include <cstdlib>

#include "sweep_common.cuh"

namespace mcinv {
namespace {

using ZW2 = ZWK<double, 2>;

// both chains' (z, w) of one row in one 256-bit load. volatile (kept in program order
// with the fences and the other volatile accesses) but without a memory clobber, so
// the plain shared-memory reads of the plan can be scheduled around it
__device__ __forceinline__ ZW2 ld_zw2(const ZW<double> *p) {
    ZW2 r;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0].z), "=d"(r.v[0].w), "=d"(r.v[1].z), "=d"(r.v[1].w)
                 : "l"(p));
    return r;
}

// diagnostic ablations (timing only, results wrong; never in the product build):
// bit 1 skip the dependency waits, bit 2 gather every neighbour from the row's own line,
// bit 4 skip the sweep-end barrier, bit 8 skip the accumulation, bit 16 later chunks re-gather
// the first entry's line (an L1 hit: the cost of a chunk without its round trip)
#ifndef MCINV_ABL
#define MCINV_ABL 0
#endif
#ifndef MCINV_V6_ACCU
#define MCINV_V6_ACCU 2  // pattern re-gather batches issued together (1: one per batch)
#endif
#ifndef MCINV_V6_OFSAHEAD
#define MCINV_V6_OFSAHEAD 1  // block offsets loaded one item ahead (0: at the item start)
#endif
#ifndef MCINV_V6_EARLY
#define MCINV_V6_EARLY 1  // first chunk's gather addresses computed before the noise (0: after the waits)
#endif
#ifndef MCINV_TRACE
#define MCINV_TRACE 0
#endif
#if MCINV_TRACE
// diagnostic build only: per warp item of CTA 0 over two steady-state sweeps, the group,
// the sweep, 7 clock64 stamps and the R row indices (tools/trace_v6.py reads the dump)
constexpr int kTrItems = 8192, kTrWords = 20;
__device__ long long g_tr[kTrItems][kTrWords];
__device__ int g_trn;
#define TR_STAMP(k) do { __syncwarp(); if (tr_on && lane == 0) trrow[2 + (k)] = clock64(); } while (0)
#else
#define TR_STAMP(k) do { } while (0)
#endif
// Eq. (4)/(5) fma chains of both chains from a staged block: entries padded by the
// host to a multiple of KU with zero coefficients on a valid column (no predicate).
// a0: the first chunk's gather addresses, computed before the noise (MCINV_V6_EARLY).
template <int KU>
__device__ __forceinline__ void row_sums2(const ZW<double> *zcol, const int *col, const ZW<double> *ab, int cnt,
                                          uint32_t zst, double (&az)[2], double (&aw)[2], const ZW<double> *const *a0,
                                          long long *trc = nullptr) {
    int first = 0;
    if (a0 && cnt > 0) {
        // the first chunk from the precomputed addresses (peeled: a shared loop body would
        // keep the other chunks' scoreboard waits on its address path)
        ZW2 v[KU];
        ZW<double> c[KU];
#pragma unroll
        for (int q = 0; q < KU; ++q) v[q] = ld_zw2(a0[q]);
#pragma unroll
        for (int q = 0; q < KU; ++q) c[q] = ab[q];
#pragma unroll
        for (int q = 0; q < KU; ++q) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                az[h] = fma(c[q].z, v[q].v[h].z, az[h]);
                aw[h] = fma(c[q].w, v[q].v[h].w, aw[h]);
            }
        }
#if MCINV_TRACE
        if (trc) {
            long long tt;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(tt) : "d"(az[0]), "d"(aw[1]) : "memory");
            trc[0] = tt;
        }
#endif
        first = KU;
    }
#if MCINV_V6_EARLY
    // the columns of chunk k + 1 are read while chunk k's gathers fly (their scoreboard is
    // then clear by the time chunk k + 1 computes its addresses)
    int jn[KU];
#pragma unroll
    for (int q = 0; q < KU; ++q) jn[q] = first < cnt ? col[first + q] : 0;
#endif
    for (int e0 = first; e0 < cnt; e0 += KU) {
        int j[KU];
        ZW2 v[KU];
        ZW<double> c[KU];
#if MCINV_V6_EARLY
#pragma unroll
        for (int q = 0; q < KU; ++q) j[q] = jn[q];
#else
#pragma unroll
        for (int q = 0; q < KU; ++q) j[q] = (MCINV_ABL & 2) ? col[0] : col[e0 + q];
#endif
        const ZW<double> *a[KU];
#pragma unroll
        for (int q = 0; q < KU; ++q) {
            a[q] = ((MCINV_ABL & 16) && a0) ? a0[0] : zrow(zcol, j[q], zst);
        }
#pragma unroll
        for (int q = 0; q < KU; ++q) {
            v[q] = ld_zw2(a[q]);
            c[q] = ab[e0 + q];
        }
#if MCINV_V6_EARLY
        if (e0 + KU < cnt) {
#pragma unroll
            for (int q = 0; q < KU; ++q) jn[q] = col[e0 + KU + q];
        }
#endif
#pragma unroll
        for (int q = 0; q < KU; ++q) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                az[h] = fma(c[q].z, v[q].v[h].z, az[h]);
                aw[h] = fma(c[q].w, v[q].v[h].w, aw[h]);
            }
        }
#if MCINV_TRACE
        if (trc && e0 / KU < 3) {
            // chunk completion (the fma consumed its loads)
            long long tt;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(tt) : "d"(az[0]), "d"(aw[1]) : "memory");
            trc[e0 / KU] = tt;
        }
#endif
    }
}

// accumulation of row i's products for the two chains of the thread (accumulate_blk with
// K = 2): the chains' products are summed in the thread, then over the P lanes of the group
// (re-gathering the lower neighbours' final values, ACCU batches per round trip, from the
// kept first-chunk addresses a0: keeping the gathered registers alive instead spills at 128
// registers, -20%)
template <int P, int V, int KU>
__device__ __forceinline__ void accumulate_blk2(const ZW<double> *zcol, uint32_t zst, int4 rec, const int *col,
                                                const int2 *pz, const double (&zi)[2], const double (&wi)[2],
                                                bool acc0, bool acc1, int lane, bool gleader, bool towner, double *sd,
                                                double *sp, bool want_diag, bool want_pat,
                                                const ZW<double> *const *a0 = nullptr) {
    const int i = rec.x;
    if (want_diag || want_pat) {
        const double d = group_sum<P>((acc0 ? zi[0] * wi[0] : 0.0) + (acc1 ? zi[1] * wi[1] : 0.0));
        if ((acc0 || acc1) && gleader) {
            if (want_diag) slot_red(sd + i, d);
            if (want_pat && rec.w >= 0) slot_red(sp + rec.w, d);
        }
    }
    if (!want_pat) return;
    const int nlow = (acc0 || acc1) ? static_cast<int>(static_cast<unsigned>(rec.z) >> 16) : 0;
    if constexpr (P == 1) {
        for (int e = 0; e < nlow; ++e) {
            const ZW2 u = ld_zw2(zrow(zcol, col[e], zst));
            const int2 z2 = pz[e];
            const double x = (acc0 ? zi[0] * u.v[0].w : 0.0) + (acc1 ? zi[1] * u.v[1].w : 0.0);
            const double y = (acc0 ? u.v[0].z * wi[0] : 0.0) + (acc1 ? u.v[1].z * wi[1] : 0.0);
            if (z2.x >= 0) slot_red(sp + z2.x, x);
            if (z2.y >= 0) slot_red(sp + z2.y, y);
        }
    } else {
        constexpr int VE = V / 2;
        const int nb = (__reduce_max_sync(0xffffffffu, nlow) + VE - 1) / VE;
#if MCINV_V6_ACCU > 1
        // the re-gathers of ACCU batches issued together (one L2 round trip for them all
        // instead of one per batch)
        constexpr int NU = MCINV_V6_ACCU;
        for (int b0 = 0; b0 < nb; b0 += NU) {
            ZW2 u[NU * VE];
            bool done_ld = false;
            if constexpr (NU * VE <= KU) {
                if (a0 && b0 == 0) {  // the lower neighbours are entries 0..: their addresses are kept
#pragma unroll
                    for (int q = 0; q < NU * VE; ++q) {
                        if (q < nlow) u[q] = ld_zw2(a0[q]);
                        else u[q] = ZW2{};
                    }
                    done_ld = true;
                }
            }
            if (!done_ld) {
                const ZW<double> *a[NU * VE];
#pragma unroll
                for (int q = 0; q < NU * VE; ++q) {
                    const int e = b0 * VE + q;
                    a[q] = zrow(zcol, e < nlow ? col[e] : 0, zst);
                        }
#pragma unroll
                for (int q = 0; q < NU * VE; ++q) {
                    const int e = b0 * VE + q;
                    if (e < nlow) u[q] = ld_zw2(a[q]);
                    else u[q] = ZW2{};
                }
            }
#pragma unroll
            for (int bb = 0; bb < NU; ++bb) {
                const int b = b0 + bb;
                if (b < nb) {
                    double v[V];
#pragma unroll
                    for (int q = 0; q < VE; ++q) {
                        const ZW2 &x2 = u[bb * VE + q];
                        v[2 * q] = (acc0 ? zi[0] * x2.v[0].w : 0.0) + (acc1 ? zi[1] * x2.v[1].w : 0.0);
                        v[2 * q + 1] = (acc0 ? x2.v[0].z * wi[0] : 0.0) + (acc1 ? x2.v[1].z * wi[1] : 0.0);
                    }
                    int held;
                    const double x = transpose_sum<P, V>(v, lane, held);
                    const int e = b * VE + (held >> 1);
                    if (towner && e < nlow) {
                        const int2 z2 = pz[e];
                        const int slot = (held & 1) ? z2.y : z2.x;
                        if (slot >= 0) slot_red(sp + slot, x);
                    }
                }
            }
        }
        return;
#endif
        for (int b = 0; b < nb; ++b) {
            double v[V];
#pragma unroll
            for (int q = 0; q < VE; ++q) {
                const int e = b * VE + q;
                const bool ok = e < nlow;
                const ZW2 u = ld_zw2(zrow(zcol, (ok ? col[e] : 0), zst));
                const double x = (acc0 ? zi[0] * u.v[0].w : 0.0) + (acc1 ? zi[1] * u.v[1].w : 0.0);
                const double y = (acc0 ? u.v[0].z * wi[0] : 0.0) + (acc1 ? u.v[1].z * wi[1] : 0.0);
                v[2 * q] = ok ? x : 0.0;
                v[2 * q + 1] = ok ? y : 0.0;
            }
            int held;
            const double x = transpose_sum<P, V>(v, lane, held);
            const int e = b * VE + (held >> 1);
            if (towner && e < nlow) {
                const int2 z2 = pz[e];
                const int slot = (held & 1) ? z2.y : z2.x;
                if (slot >= 0) slot_red(sp + slot, x);
            }
        }
    }
}

}  // namespace

// BITS: one completion bit per row (see sweep5_kernel); GAUSS: compile-time Gaussian noise
template <int KU, int NT, int LGC, int LGP, bool BITS, bool GAUSS>
__global__ void __launch_bounds__(NT, 1) sweep6_kernel(const Sweep3Params<double> p) {
    const uint32_t zst = static_cast<uint32_t>(p.ld) * static_cast<uint32_t>(sizeof(ZW<double>));
    constexpr int P = 1 << LGP;  // lanes of one SE group in a row (2 chains each)
    constexpr int V = P < 8 ? P : 8;
    constexpr int C = 1 << LGC;  // chains per CTA
    constexpr int LR = C / 2;    // lanes per row
    constexpr int R = 32 / LR;   // rows per warp group
    extern __shared__ __align__(128) unsigned char sm6[];
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    const int W = B >> 5;
    const int w = tid >> 5;
    const int lane = tid & 31;
    const int cl = lane & (LR - 1);
    const int chain = (blockIdx.x << LGC) + 2 * cl;  // the thread's chains: chain, chain + 1
    const bool active0 = chain < p.chains, active1 = chain + 1 < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);  // even (chain_begin % group_size == 0)
    const bool gleader = (cl & (P - 1)) == 0;
    const bool towner = (lane & ((P > V ? P / V : 1) - 1)) == 0;
    const int64_t grp = chain >> p.lgG;
    ZW<double> *__restrict__ zcol = p.zw + chain;
    const bool want_diag = p.outputs & OUT_DIAG, want_pat = p.outputs & OUT_PATTERN;
    const bool want_full = p.outputs & OUT_FULL;
    double *const sd = p.slot_diag + grp * p.n;
    double *const sp = p.slot_pat + grp * p.pcount;
    // shared memory: [W][2] mbarriers | [W][2][maxb] block slots | done[n]
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm6);
    unsigned char *blk = sm6 + 16 * W;
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

    const int ngroups = p.nslots / R;
    const int sub = lane / LR;
    auto issue = [&](int g, unsigned char *dst, uint32_t bar) {
        const int64_t off = __ldg(p.gofs + g);
        const uint32_t bytes = static_cast<uint32_t>(__ldg(p.gofs + g + 1) - off);
        tma_block(smem_addr(dst), p.blob + off, bytes, bar);
    };
    if (lane == 0 && w < ngroups) issue(w, buf0, bar0);
#if MCINV_V6_OFSAHEAD
    // lane 0 holds the block offsets of the group it stages next, loaded one item ahead (the
    // __ldg of gofs no longer sits between an item's start and its TMA issue)
    int64_t nx_off = 0, nx_end = 0;
    if (lane == 0 && w < ngroups) {
        const int g1 = w + W < ngroups ? w + W : w;
        nx_off = __ldg(p.gofs + g1);
        nx_end = __ldg(p.gofs + g1 + 1);
    }
#endif
    uint32_t ph0 = 0, ph1 = 0;
    int item = 0;
    bool dv = false;  // divergence seen (reading R12)
    for (int s = p.s_begin; s < p.s_end; ++s) {
        const uint32_t k = p.sweep_abs0 + static_cast<uint32_t>(s);
        const bool sampling = s >= p.burn_in;
        const unsigned char need = static_cast<unsigned char>(s + 1);
        for (int g = w; g < ngroups; g += W, ++item) {
            const bool odd = item & 1;
            unsigned char *cur = odd ? buf1 : buf0;
            // stage the next item's block into the other slot (its previous item is done)
            const int gn = g + W < ngroups ? g + W : w;
            const bool has_next = g + W < ngroups || s + 1 < p.s_end;
#if MCINV_TRACE
            const bool tr_on = blockIdx.x == 0 && s >= p.s_begin + 20 && s < p.s_begin + 22;
            long long *trrow = nullptr;
            if (tr_on) {
                int slot = 0;
                if (lane == 0) slot = atomicAdd(&g_trn, 1);
                slot = __shfl_sync(0xffffffffu, slot, 0);
                trrow = g_tr[slot < kTrItems ? slot : kTrItems - 1];
                if (lane == 0) { trrow[0] = g; trrow[1] = s; }
            }
            TR_STAMP(0);
#endif
#if MCINV_V6_OFSAHEAD
            if (lane == 0 && has_next) {
                tma_block(smem_addr(odd ? buf0 : buf1), p.blob + nx_off, static_cast<uint32_t>(nx_end - nx_off),
                          odd ? bar0 : bar1);
                const int g2 = gn + W < ngroups ? gn + W : w;
                nx_off = __ldg(p.gofs + g2);
                nx_end = __ldg(p.gofs + g2 + 1);
            }
#else
            if (lane == 0 && has_next) issue(gn, odd ? buf0 : buf1, odd ? bar0 : bar1);
#endif
            if (odd) {
                mbar_wait(bar1, ph1);
                ph1 ^= 1;
            } else {
                mbar_wait(bar0, ph0);
                ph0 ^= 1;
            }
            // block: head | rec[R] | dsg[R][2] | wait masks[R] (16-B padded) | col | ab | pz
            constexpr int kMaskBytes = (4 * R + 15) / 16 * 16;
            const int4 head = reinterpret_cast<const int4 *>(cur)[0];
            const int4 rec = reinterpret_cast<const int4 *>(cur)[1 + sub];
            const unsigned wmask = reinterpret_cast<const unsigned *>(cur + 16 + 32 * R)[sub];
            const int *col = reinterpret_cast<const int *>(cur + 16 + 32 * R + kMaskBytes) + rec.y;
            const ZW<double> *ab = reinterpret_cast<const ZW<double> *>(cur + head.z) + rec.y;
            const int2 *pz = reinterpret_cast<const int2 *>(cur + head.w) + rec.y;
            const double *dsg = reinterpret_cast<const double *>(cur + 16 + 16 * R) + 2 * sub;
            const bool valid = rec.x >= 0;
            const int i = rec.x, cnt = valid ? rec.z & 0xffff : 0;
#if MCINV_TRACE
            TR_STAMP(1);
            if (tr_on && cl == 0 && sub < 8) trrow[9 + sub] = i;
            if (tr_on && lane == 0) trrow[17] = trrow[18] = trrow[19] = 0;
#endif
            double zi[2] = {0.0, 0.0}, wi[2] = {0.0, 0.0};
            double phi0 = 0.0, phi1 = 0.0;
#if MCINV_V6_EARLY
            // the first chunk's gather addresses, computed with the prefetches (before the noise
            // and the waits) and kept opaque in registers: the gathers then issue back to back
            // once the waits pass. Computed after the waits, ptxas put the column reads (shared
            // loads) on the scoreboard of the first gathers, so the fifth address waited for the
            // first gather's round trip: every chunk took two (ncu + SASS control bits;
            // config 2 +4.5%, profiles/r02_v6_early.log)
            const ZW<double> *a0[KU];
#pragma unroll
            for (int q = 0; q < KU; ++q) a0[q] = zcol;
            const ZW<double> *const *a0p = a0;
#else
            const ZW<double> *const *a0p = nullptr;
#endif
            if (valid) {
                const int nlow = static_cast<int>(static_cast<unsigned>(rec.z) >> 16);
#if MCINV_V6_EARLY
                if (cnt > 0) {
#pragma unroll
                    for (int q = 0; q < KU; ++q) {
                        a0[q] = zrow(zcol, col[q], zst);
                        asm volatile("" : "+l"(a0[q]));  // opaque: kept in registers, not recomputed later
                        if (p.prefetch >= 2) prefetch_l2(a0[q]);
                    }
                }
                if (p.prefetch & 8) {
                    // the later chunks' lines with an L1 prefetch (measured +1%, profiles/r02_v6_stage.log)
                    for (int e0 = KU; e0 < cnt; e0 += KU)
#pragma unroll
                        for (int q = 0; q < KU; ++q) prefetch_l1(zrow(zcol, col[e0 + q], zst));
                } else if (p.prefetch >= 2) {
                    for (int e0 = KU; e0 < cnt; e0 += KU)
#pragma unroll
                        for (int q = 0; q < KU; ++q) prefetch_l2(zrow(zcol, col[e0 + q], zst));
                } else
#endif
                // every neighbour's line on its way into L2 while the noise runs
                if (p.prefetch == 1) {  // into L1 (the SM's own L1 sees its CTA's stores)
                    for (int e0 = 0; e0 < cnt; e0 += KU)
#pragma unroll
                        for (int q = 0; q < KU; ++q) prefetch_l1(zrow(zcol, col[e0 + q], zst));
                } else if (p.prefetch) {
                    for (int e0 = 0; e0 < cnt; e0 += KU)
#pragma unroll
                        for (int q = 0; q < KU; ++q) prefetch_l2(zrow(zcol, col[e0 + q], zst));
                }
                // the pair's noise: one Philox block, ln and sqrt for both chains (reading R4)
                if constexpr (GAUSS) {
                    gaussian2(static_cast<uint32_t>(i), k, gchain, p.key0, p.key1, phi0, phi1);
                } else {
                    phi0 = noise_phi(p.noise, static_cast<uint32_t>(i), k, gchain, p.key0, p.key1);
                    phi1 = noise_phi(p.noise, static_cast<uint32_t>(i), k, gchain + 1u, p.key0, p.key1);
                }
                // the upper neighbours' lines (previous sweep's values: stable until this row
                // publishes) into L1 right before the waits, so that the chunks after the first
                // hit L1 once the lower neighbours are final
                if (p.prefetch & 4) {
                    for (int e = nlow; e < cnt; ++e) prefetch_l1(zrow(zcol, col[e], zst));
                }
#if MCINV_TRACE
            }
            TR_STAMP(2);
            if (valid) {
                const int nlow = static_cast<int>(static_cast<unsigned>(rec.z) >> 16);
                auto wait_on = [&](int j) {
                    auto ready = [&]() -> bool {
                        if constexpr (BITS)
                            return ((reinterpret_cast<volatile unsigned *>(dbits)[j >> 5] >> (j & 31)) & 1u) ==
                                   (need & 1u);
                        else
                            return reinterpret_cast<volatile unsigned char *>(done)[j] == need;
                    };
                    wait_ready(ready, p.err, 0);
                };
                for (unsigned m = wmask; m; m &= m - 1) wait_on(col[__ffs(m) - 1]);
                for (int e = 32; e < nlow; ++e) wait_on(col[e]);
            }
            TR_STAMP(3);
            if (false) {
                const int nlow = 0;
#endif
                // lower neighbours whose completion is not implied (the host's wait mask;
                // entries from 32 on always)
                auto wait_on = [&](int j) {
                    auto ready = [&]() -> bool {
                        if constexpr (BITS)
                            return ((reinterpret_cast<volatile unsigned *>(dbits)[j >> 5] >> (j & 31)) & 1u) ==
                                   (need & 1u);
                        else
                            return reinterpret_cast<volatile unsigned char *>(done)[j] == need;
                    };
                    wait_ready(ready, p.err, 0);
                };
                if (!(MCINV_ABL & 1)) {
                    for (unsigned m = wmask; m; m &= m - 1) wait_on(col[__ffs(m) - 1]);
                    for (int e = 32; e < nlow; ++e) wait_on(col[e]);
                }
            }
            if (valid) {
                __threadfence_block();  // acquire
                double az[2] = {0.0, 0.0}, aw[2] = {0.0, 0.0};
#if MCINV_TRACE
                row_sums2<KU>(zcol, col, ab, cnt, zst, az, aw, a0p, (tr_on && lane == 0) ? trrow + 17 : nullptr);
#else
                row_sums2<KU>(zcol, col, ab, cnt, zst, az, aw, a0p);
#endif
                const double dl = dsg[0], sg = dsg[1];
                zi[0] = fma(-dl, az[0], sg * phi0);
                wi[0] = fma(-dl, aw[0], sg * phi0);
                zi[1] = fma(-dl, az[1], sg * phi1);
                wi[1] = fma(-dl, aw[1], sg * phi1);
                st256(zrow(zcol, i, zst), zi[0], wi[0], zi[1], wi[1]);
                dv = dv | (active0 & (bad_s(zi[0]) | bad_s(wi[0]))) | (active1 & (bad_s(zi[1]) | bad_s(wi[1])));
                if (want_full && sampling) {
                    const int64_t ts = s - p.snap_s0;
                    p.snap_x[(ts * p.n + i) * p.ld + chain] = zi[0];
                    p.snap_y[(ts * p.n + i) * p.ld + chain] = wi[0];
                    p.snap_x[(ts * p.n + i) * p.ld + chain + 1] = zi[1];
                    p.snap_y[(ts * p.n + i) * p.ld + chain + 1] = wi[1];
                }
            }
            TR_STAMP(4);
            __syncwarp();  // the row's stores are ordered before its counter update
            if (valid && cl == 0) {
                if constexpr (BITS) {
                    __threadfence_block();  // release
                    atomicXor(dbits + (i >> 5), 1u << (i & 31));
                } else {
                    const unsigned short vv = need;
                    asm volatile("st.release.cta.shared::cta.u8 [%0], %1;" ::"r"(smem_addr(done + i)), "h"(vv)
                                 : "memory");
                }
            }
            TR_STAMP(5);
            if (sampling && !(MCINV_ABL & 8)) {
                    accumulate_blk2<P, V, KU>(zcol, zst, rec, col, pz, zi, wi, valid && active0, valid && active1, lane,
                                          gleader, towner, sd, sp, want_diag, want_pat, a0p);
            }
            __syncwarp();  // reconverge; orders this item's block reads before the next TMA into it
            TR_STAMP(6);
        }
        if (!(MCINV_ABL & 4)) __syncthreads();  // sweep boundary: all reads of sweep s values are done
    }
    if (dv) atomicAdd(p.bad, 1.0);
}

namespace {

#ifndef MCINV_V6_KU768
#define MCINV_V6_KU768 2
#endif
// gathers in flight per thread at 512 threads; config 2: KU 4 2.53e10, 5 2.61e10, 6 2.65e10,
// 7 2.47e10, 8 2.41e10 site-updates/s (profiles/r02_v6_ku512.log)
#ifndef MCINV_V6_KU512
#define MCINV_V6_KU512 6
#endif
template <int NT, int LGC, int LGP, bool BITS>
cudaError_t launch6b(const Sweep3Params<double> &p, int threads, cudaStream_t st) {
    // gathers in flight: 64 registers at 1024 threads, 85 at 768, 128 at 512 (KU = 6: 128 registers, no spill)
    constexpr int KU = NT > 768 ? 2 : NT > 512 ? MCINV_V6_KU768 : MCINV_V6_KU512;
    if (threads > NT) return cudaErrorInvalidConfiguration;
    const int blocks = (p.chains + (1 << LGC) - 1) >> LGC;
    const size_t smem = sweep6_smem(p.n, threads, p.maxb);
    auto k = p.noise == 0 ? sweep6_kernel<KU, NT, LGC, LGP, BITS, true> : sweep6_kernel<KU, NT, LGC, LGP, BITS, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int carve = (int)((smem + 8192) * 100 / (228 * 1024)) + 1;
    if (const char *ev = std::getenv("MCINV_CARVE")) carve = std::atoi(ev);
    if (carve >= 0) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve > 100 ? 100 : carve);
        if (e != cudaSuccess) return e;
    }
    k<<<blocks, threads, smem, st>>>(p);
    return cudaGetLastError();
}

template <int LGC, int LGP>
cudaError_t launch6(const Sweep3Params<double> &p, int threads, cudaStream_t st) {
    if constexpr (LGP > LGC - 1 || LGC < 1) {
        return cudaErrorInvalidValue;
    } else {
        const bool bits = p.n > kByteCounters;
        if (threads > 768)
            return bits ? launch6b<1024, LGC, LGP, true>(p, threads, st) : launch6b<1024, LGC, LGP, false>(p, threads, st);
        if (threads > 512)
            return bits ? launch6b<768, LGC, LGP, true>(p, threads, st) : launch6b<768, LGC, LGP, false>(p, threads, st);
        return bits ? launch6b<512, LGC, LGP, true>(p, threads, st) : launch6b<512, LGC, LGP, false>(p, threads, st);
    }
}

template <int LGC>
cudaError_t launch6c(const Sweep3Params<double> &p, int threads, cudaStream_t st) {
    switch (p.lgP) {  // lanes of a group per row: log2(min(group size, C) / 2)
        case 0: return launch6<LGC, 0>(p, threads, st);
        case 1: return launch6<LGC, 1>(p, threads, st);
        case 2: return launch6<LGC, 2>(p, threads, st);
        case 3: return launch6<LGC, 3>(p, threads, st);
        case 4: return launch6<LGC, 4>(p, threads, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

#if MCINV_TRACE
extern "C" int mcinv_debug_trace_dump(const char *path) {
    static long long h[kTrItems][kTrWords];
    int nn = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_tr, sizeof(h));
    cudaMemcpyFromSymbol(&nn, g_trn, sizeof(int));
    FILE *f = fopen(path, "wb");
    if (!f) return -1;
    if (nn > kTrItems) nn = kTrItems;
    fwrite(h, sizeof(long long) * kTrWords, nn, f);
    fclose(f);
    return nn;
}
#endif

size_t sweep6_smem(int n, int threads, int maxb) {
    const size_t W = (size_t)threads / 32;
    const size_t counters = n > kByteCounters ? ((size_t)n + 127) / 128 * 16 : ((size_t)n + 15) / 16 * 16;
    return 16 * W + 2 * W * (size_t)maxb + counters;
}

int sweep6_ku(int threads) { return threads > 768 ? 2 : threads > 512 ? MCINV_V6_KU768 : MCINV_V6_KU512; }

cudaError_t launch_sweep6(const Sweep3Params<double> &p, int threads, cudaStream_t st) {
    switch (p.lgC) {
        case 1: return launch6c<1>(p, threads, st);
        case 2: return launch6c<2>(p, threads, st);
        case 3: return launch6c<3>(p, threads, st);
        case 4: return launch6c<4>(p, threads, st);
        case 5: return launch6c<5>(p, threads, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mcinv
