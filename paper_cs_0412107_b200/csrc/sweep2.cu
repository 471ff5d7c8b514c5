// sweep2.cu -- K1/K2 (v2): the CC sweep on a dependency-respecting step
// schedule (plan.h), warp-specialized.
//
// One CTA owns C chains; lanes = C chains x R row slots (C * R = 32). The
// planner guarantees that the rows of a step do not depend on each other and
// that every operand is exactly the one the sequential sweep (Eq. 4/5,
// PAPER.md:157-160) reads, so z and w are bit-identical to row-by-row order.
//
// Warp roles (all synchronised with mbarriers, per step slot):
//   A  (1 warp)   the serial part: for each step, the fma chains of
//                 Eq. (4)/(5) over smem operands, z_i, w_i to HBM and to the
//                 16-step result ring, FULL-output snapshots, staging.
//   B  (1 warp)   producer: TMA bulk copy of the record tile of step U+8
//                 (cols, coefficients, smem source offsets, accumulation
//                 records) and cp.async gathers of step U's far operands
//                 (>= 8 steps old) from the [n][ld] state in HBM; waits only
//                 for A (step U-7 done).
//   D  (ND warps) accumulation (sampling sweeps): A stages each finished
//                 row's z_i, w_i and its partner values; D forms the diag and
//                 pattern products (Eq. 1/C), sums them over the
//                 chains of an SE group and does one RMW (or RED) per group
//                 slot. The trace w^dagger Q z (Eq. tr) is summed
//                 in A's registers.
//   N  (NW warps) noise: phi(row, sweep, chain) by Philox4x32-10 + Box-Muller
//                 (noise.cuh) into an smem ring, round-robin over steps.
// A and B are single warps; N and D are NW / ND warps taking steps in turn.
#include "mcinv_internal.cuh"
#include "noise.cuh"
#include "plan.h"
#include "scalar.cuh"

namespace mcinv {

namespace {

constexpr int NQ = 8;  // noise ring slots

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ uint32_t mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Blocking wait with a watchdog: a protocol bug traps after 20 s instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    const uint64_t t0 = globaltimer_ns();
    while (!mbar_try(bar, parity))
        if (globaltimer_ns() - t0 > 20000000000ull) __trap();
}
// non-blocking probe of a phase (result consumed later: hides the latency)
__device__ __forceinline__ uint32_t mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// arrive on the mbarrier when all prior cp.async of this thread complete
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

template <typename S>
__device__ __forceinline__ S lds_s(const unsigned char *p) {
    return *reinterpret_cast<const S *>(p);
}

// phase parity of the u-th use of a step-indexed barrier slot (u = (T - T0) / nslots)
template <int NSLOTS>
__device__ __forceinline__ uint32_t par(uint32_t T, uint32_t T0) {
    return ((T - T0) / NSLOTS) & 1u;
}

}  // namespace

// Stage slot (A -> D): int P; int2 ids[P+1][R] ({pzi, pzo} per partner record,
// {dslot, pslot} for the row itself at index P); ZW vals[P+1][32] (partner
// values per lane, the row's own z_i, w_i at index P).
__host__ __device__ constexpr int stage_ids_off() { return 16; }
template <int ESZ>
__host__ __device__ inline int stage_vals_off(int max_parts, int R) {
    return (16 + 8 * (max_parts + 1) * R + 15) & ~15;
}
template <int ESZ>
__host__ __device__ inline int stage_slot_bytes(int max_parts, int R) {
    return stage_vals_off<ESZ>(max_parts, R) + (max_parts + 1) * 32 * 2 * ESZ;
}
constexpr int NSTG = 4;  // stage slots

// Warp roles: 0 = A; 1..NW = N; NW+1 = B; NW+2 .. NW+1+ND = D. Warps share an
// SMSP by index mod 4, so A pairs with B and each D with a noise warp.
template <typename S, int C, int R, int NW, int ND>
__global__ void __launch_bounds__(32 * (2 + NW + ND)) sweep2_kernel(const Sweep2Params<S> p) {
    constexpr int ESZ = sizeof(S);
    constexpr int ZWSZ = 2 * ESZ;
    using VA = ValueArea<ESZ>;
    constexpr int BLK = VA::BLK;
    constexpr int WB = NW + 1;  // producer warp

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *vals = smem;
    unsigned char *tiles = smem + VA::BYTES;
    double *noise = reinterpret_cast<double *>(tiles + NTILE * p.tile_slot);   // [NQ][32]
    unsigned char *stage0 = reinterpret_cast<unsigned char *>(noise + NQ * 32);  // [NSTG] stage slots
    const int stg_bytes = stage_slot_bytes<ESZ>(p.max_items, R);
    const int stg_vals = stage_vals_off<ESZ>(p.max_items, R);
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage0 + (size_t)NSTG * stg_bytes);
    const uint32_t b_tile = smem_u32(bars);               // [NTILE] TMA complete_tx
    const uint32_t b_gather = b_tile + 8 * NTILE;         // [NGBUF] 32 cp.async arrivals
    const uint32_t b_adone = b_gather + 8 * NGBUF;        // [NGBUF] A finished step
    const uint32_t b_sfull = b_adone + 8 * NGBUF;         // [NSTG] stage written
    const uint32_t b_sempty = b_sfull + 8 * NSTG;         // [NSTG] stage reduced
    const uint32_t b_nfull = b_sempty + 8 * NSTG;         // [NQ] noise ready
    const uint32_t b_nempty = b_nfull + 8 * NQ;           // [NQ] noise consumed

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = lane % C, r = lane / C;
    const int cb = blockIdx.x * C;
    const int chain = cb + c;
    const bool active = chain < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);
    const int coff = c * ZWSZ;
    const int roff = r * C * ZWSZ;
    const uint32_t S_n = (uint32_t)p.steps;
    const uint32_t T0 = (uint32_t)p.s_begin * S_n, T_end = (uint32_t)p.s_end * S_n;
    // first sampling step: the stage ring (A -> D) counts its phases from here
    const uint32_t Ts = max(T0, (uint32_t)p.burn_in * S_n);
    const uint32_t tile_slot = (uint32_t)p.tile_slot;
    const bool want_tr = (p.outputs & OUT_TRACE) != 0;
    const bool want_red = (p.outputs & (OUT_DIAG | OUT_PATTERN)) != 0;
    auto tile_of = [&](uint32_t T) { return tiles + (T % NTILE) * tile_slot; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NTILE; ++s) mbar_init(b_tile + 8 * s, 1);
        for (int s = 0; s < NGBUF; ++s) {
            mbar_init(b_gather + 8 * s, 32);
            mbar_init(b_adone + 8 * s, 1);
        }
        for (int s = 0; s < NSTG; ++s) {
            mbar_init(b_sfull + 8 * s, 1);
            mbar_init(b_sempty + 8 * s, 1);
        }
        for (int s = 0; s < NQ; ++s) {
            mbar_init(b_nfull + 8 * s, 1);
            mbar_init(b_nempty + 8 * s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        // zero block and the ring of the 7 steps before T0 (from the state)
        for (int b = lane; b < BLK / 16; b += 32)
            reinterpret_cast<double2 *>(vals + VA::ZERO)[b] = make_double2(0.0, 0.0);
        for (int q = 1; q <= PDIST; ++q) {
            const int64_t T = (int64_t)T0 - q;
            const int t = (int)(((T % (int64_t)S_n) + S_n) % S_n);
            const int *g = reinterpret_cast<const int *>(p.tiles + p.tile_off[t] + 32);
            const int row = g[r], flg = g[R + r];
            if (row >= 0 && (flg & 2))
                *reinterpret_cast<ZW<S> *>(vals + (((T % NRING) + NRING) % NRING) * BLK + roff + coff) =
                    p.zw[(int64_t)row * p.ld + chain];
        }
    }
    __syncthreads();

    if (warp == WB) {
        // ================= B: tiles and gathers (waits only for A)
        const unsigned char *zw_chain = reinterpret_cast<const unsigned char *>(p.zw + chain);
        const int64_t row_bytes = (int64_t)p.ld * ZWSZ;
        const unsigned char *gtiles = p.tiles;
        const uint32_t vbase = smem_u32(vals) + coff;
        if (lane == 0)
            for (uint32_t T = T0; T < T0 + 8 && T < T_end; ++T) {
                const int t = (int)(T % S_n);
                tma_load_1d(smem_u32(tile_of(T)), gtiles + p.tile_off[t], (uint32_t)(p.tile_off[t + 1] - p.tile_off[t]),
                            b_tile + 8 * (T % NTILE));
            }
        for (uint32_t U = T0; U < T_end; ++U) {
            // gather slot U % 8 was used by step U-8 and, for partners of a
            // row's previous segment, by step U-7: wait for A to finish U-7
            if (U >= T0 + 7) mbar_wait(b_adone + 8 * ((U - 7) % NGBUF), par<NGBUF>(U - 7, T0));
            mbar_wait(b_tile + 8 * (U % NTILE), par<NTILE>(U, T0));
            const unsigned char *tl = tile_of(U);
            const int K = reinterpret_cast<const int *>(tl)[0];
            if (lane == 0 && U + 8 < T_end) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_load_1d(smem_u32(tile_of(U + 8)), gtiles + *reinterpret_cast<const int64_t *>(tl + 16),
                            (uint32_t)reinterpret_cast<const int *>(tl)[2], b_tile + 8 * ((U + 8) % NTILE));
            }
            const int2 *meta = reinterpret_cast<const int2 *>(tl + TileLayout{0, 0, R, ESZ}.meta()) + r;
            for (int k = 0; k < K; ++k) {
                const int2 m = meta[k * R];
                if (m.y >= 0) {
                    const unsigned char *src = zw_chain + (int64_t)m.y * row_bytes;
                    const uint32_t dst = vbase + m.x;
#pragma unroll
                    for (int h = 0; h < ZWSZ / 16; ++h) cp_async16(dst + 16 * h, src + 16 * h);
                }
            }
            cp_async_arrive(b_gather + 8 * (U % NGBUF));
        }
    } else if (warp == 0) {
        // ================= A: the serial fma chains, then stage the row's accumulation operands
        S acc_z = zero_s<S>(), acc_w = zero_s<S>(), tr = zero_s<S>();
        ZW<S> *zw_chain = p.zw + chain;
        const unsigned char *vlane = vals + coff;
        unsigned char *ring_lane = vals + roff + coff;
        const bool stage_on = want_red || want_tr;
        uint32_t ok_g = 0, ok_n = 0, ok_s = 0;
        for (uint32_t T = T0; T < T_end; ++T) {
            if (!ok_g) mbar_wait(b_gather + 8 * (T % NGBUF), par<NGBUF>(T, T0));
            const unsigned char *tl = tile_of(T);
            const int K = reinterpret_cast<const int *>(tl)[0];
            const int P = reinterpret_cast<const int *>(tl)[1];
            const TileLayout L{K, P, R, ESZ};
            const int flags = reinterpret_cast<const int *>(tl + 32)[R + r];
            if (flags & 1) {
                acc_z = zero_s<S>();
                acc_w = zero_s<S>();
            }
            const int2 *meta = reinterpret_cast<const int2 *>(tl + L.meta()) + r;
            const unsigned char *cf = tl + L.coef() + 2 * ESZ * r;
            for (int k = 0; k < K; ++k) {
                const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vlane + meta[k * R].x);
                acc_z = fma_s(lds_s<S>(cf + 2 * ESZ * R * k), v.z, acc_z);
                acc_w = fma_s(lds_s<S>(cf + 2 * ESZ * R * k + ESZ), v.w, acc_w);
            }
            // probe the next step's barriers while the fma chains drain
            const uint32_t Tn = T + 1;
            ok_g = Tn < T_end ? mbar_test(b_gather + 8 * (Tn % NGBUF), par<NGBUF>(Tn, T0)) : 1u;
            if (!ok_n) mbar_wait(b_nfull + 8 * (T % NQ), par<NQ>(T, T0));
            const uint32_t s_loc = T / S_n;
            const bool sampling = (int)s_loc >= p.burn_in;
            S zi = zero_s<S>(), wi = zero_s<S>();
            const bool last = (flags & 2) != 0;
            if (last) {
                const int row = reinterpret_cast<const int *>(tl + 32)[r];
                const double phi = noise[(T % NQ) * 32 + lane];
                const S dl = lds_s<S>(tl + L.dsq() + r * ESZ);
                const S sg = lds_s<S>(tl + L.dsq() + (R + r) * ESZ);
                zi = fma_s(neg_s(dl), acc_z, scale_s(sg, phi));
                wi = fma_s(neg_s(conj_s(dl)), acc_w, scale_s(conj_s(sg), phi));
                zw_chain[(int64_t)row * p.ld] = ZW<S>{zi, wi};
                *reinterpret_cast<ZW<S> *>(ring_lane + (T % NRING) * BLK) = ZW<S>{zi, wi};
                if ((p.outputs & OUT_FULL) && sampling) {
                    const int64_t t = (int64_t)s_loc - p.snap_s0;
                    p.snap_x[(t * p.n + row) * p.ld + chain] = zi;
                    p.snap_y[(t * p.n + row) * p.ld + chain] = wi;
                }
            }
            ok_n = Tn < T_end ? mbar_test(b_nfull + 8 * (Tn % NQ), par<NQ>(Tn, T0)) : 1u;
            if (stage_on && sampling) {
                // partner values and slot ids of the finished rows -> stage slot (D reduces)
                if (!ok_s && T >= Ts + NSTG) mbar_wait(b_sempty + 8 * (T % NSTG), par<NSTG>(T - NSTG, Ts));
                unsigned char *sg_ = stage0 + (T % NSTG) * stg_bytes;
                int2 *ids = reinterpret_cast<int2 *>(sg_ + stage_ids_off()) + r;
                unsigned char *sv = sg_ + stg_vals + lane * ZWSZ;
                const int *rs = reinterpret_cast<const int *>(tl + 32);
                const bool live = last && active;
                S qz = mul_s(lds_s<S>(tl + L.dsq() + (2 * R + r) * ESZ), zi);
                S qw = zero_s<S>();
                const unsigned char *pr = tl + L.part() + L.part_bytes() * r;
                for (int q = 0; q < P; ++q, pr += L.part_bytes() * R) {
                    const int4 rec = *reinterpret_cast<const int4 *>(pr);
                    const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vlane + rec.x);
                    *reinterpret_cast<ZW<S> *>(sv + q * 32 * ZWSZ) = v;
                    if (c == 0) ids[q * R] = last ? make_int2(rec.y, rec.z) : make_int2(-1, -1);
                    if (want_tr) {
                        qz = add_s(qz, mul_s(lds_s<S>(pr + 16), v.z));
                        qw = add_s(qw, mul_s(lds_s<S>(pr + 16 + ESZ), conj_s(v.w)));
                    }
                }
                *reinterpret_cast<ZW<S> *>(sv + P * 32 * ZWSZ) = ZW<S>{zi, wi};
                if (c == 0) ids[P * R] = last ? make_int2(rs[2 * R + r], rs[3 * R + r]) : make_int2(-1, -1);
                if (lane == 0) reinterpret_cast<int *>(sg_)[0] = P;
                if (want_tr && live) tr = add_s(tr, add_s(zwc_s(qz, wi), mul_s(zi, qw)));
                __syncwarp();
                if (lane == 0) mbar_arrive(b_sfull + 8 * (T % NSTG));
                ok_s = (Tn < T_end && Tn >= Ts + NSTG) ? mbar_test(b_sempty + 8 * (Tn % NSTG), par<NSTG>(Tn - NSTG, Ts))
                                                       : 1u;
            } else {
                __syncwarp();
                ok_s = 0;
            }
            if (lane == 0) {
                mbar_arrive(b_nempty + 8 * (T % NQ));
                mbar_arrive(b_adone + 8 * (T % NGBUF));
            }
        }
        if (want_tr) {
            // trace: sum over the row slots and the chains of each SE group, one atomic per group part
            const int gse = p.gs < C ? p.gs : C;
            S v = active ? tr : zero_s<S>();
            for (int off = C; off < 32; off <<= 1) v = add_s(v, shfl_xor_s(v, off));
            for (int off = 1; off < gse; off <<= 1) v = add_s(v, shfl_xor_s(v, off));
            if (r == 0 && (c % gse) == 0 && active)
                atomic_add_to(p.slot_trace + (int64_t)((cb + c) / p.gs) * (ESZ / 8), v);
        }
    } else if (warp > WB) {
        // ================= D: group reductions of the staged products, steps T0 + dw, T0 + dw + ND, ...
        if (want_red) {
            const int dw = warp - WB - 1;
            const int gse = p.gs < C ? p.gs : C;
            const int lg_gse = __ffs(gse) - 1;
            const int lg_tpr = 5 - lg_gse;          // tasks per (record, role): 32 / gse
            const int lg_gpr = __ffs(C / gse) - 1;  // group parts per row slot
            const bool use_atomic = p.gs > C || ND > 1;
            for (uint32_t T = Ts + dw; T < T_end; T += ND) {
                mbar_wait(b_sfull + 8 * (T % NSTG), par<NSTG>(T, Ts));
                const unsigned char *sg_ = stage0 + (T % NSTG) * stg_bytes;
                const int P = reinterpret_cast<const int *>(sg_)[0];
                const int2 *ids = reinterpret_cast<const int2 *>(sg_ + stage_ids_off());
                const ZW<S> *sv = reinterpret_cast<const ZW<S> *>(sg_ + stg_vals);
                // task = (record q, role h, row slot r2, group part g2)
                const int nt = (2 * P + 2) << lg_tpr;
                for (int tk = lane; tk < nt; tk += 32) {
                    const int qh = tk >> lg_tpr, rem = tk & ((1 << lg_tpr) - 1);
                    const int q = qh >> 1, h = qh & 1;
                    const int r2 = rem >> lg_gpr, g2 = rem & ((1 << lg_gpr) - 1);
                    const int2 id = ids[q * R + r2];
                    const int slot = h ? id.y : id.x;
                    const int c0 = g2 << lg_gse;
                    if (slot < 0 || cb + c0 >= p.chains) continue;
                    const ZW<S> *me = sv + P * 32 + r2 * C + c0;
                    const ZW<S> *pv = sv + q * 32 + r2 * C + c0;
                    S sum = zero_s<S>();
                    if (q == P) {
                        for (int cc = 0; cc < gse; ++cc) sum = add_s(sum, zwc_s(me[cc].z, me[cc].w));
                    } else if (h == 0) {
                        for (int cc = 0; cc < gse; ++cc) sum = add_s(sum, zwc_s(me[cc].z, pv[cc].w));
                    } else {
                        for (int cc = 0; cc < gse; ++cc) sum = add_s(sum, zwc_s(pv[cc].z, me[cc].w));
                    }
                    const bool to_diag = q == P && h == 0;
                    double *dst = (to_diag ? p.slot_diag + (((int64_t)(cb + c0) / p.gs) * p.n + slot) * (ESZ / 8)
                                           : p.slot_pat + (((int64_t)(cb + c0) / p.gs) * p.pcount + slot) * (ESZ / 8));
                    if (use_atomic) atomic_add_to(dst, sum);
                    else add_to(dst, sum);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(b_sempty + 8 * (T % NSTG));
            }
        } else if (want_tr) {
            // trace only: keep the stage ring turning
            const int dw = warp - WB - 1;
            for (uint32_t T = Ts + dw; T < T_end; T += ND) {
                mbar_wait(b_sfull + 8 * (T % NSTG), par<NSTG>(T, Ts));
                __syncwarp();
                if (lane == 0) mbar_arrive(b_sempty + 8 * (T % NSTG));
            }
        }
    } else {
        // ================= N: noise, steps T0 + w, T0 + w + NW, ...
        const int w = warp - 1;
        for (uint32_t T = T0 + w; T < T_end; T += NW) {
            if (T >= T0 + NQ) mbar_wait(b_nempty + 8 * (T % NQ), par<NQ>(T - NQ, T0));
            mbar_wait(b_tile + 8 * (T % NTILE), par<NTILE>(T, T0));
            const int *rs = reinterpret_cast<const int *>(tile_of(T) + 32);
            double phi = 0.0;
            if (rs[R + r] & 2) {
                if (p.noise == 0)
                    phi = gaussian(static_cast<uint32_t>(rs[r]), p.sweep_abs0 + T / S_n, gchain, p.key0, p.key1);
                else
                    phi = p.noise == 2 ? 1.0 : 0.0;
            }
            noise[(T % NQ) * 32 + lane] = phi;
            __syncwarp();
            if (lane == 0) mbar_arrive(b_nfull + 8 * (T % NQ));
        }
    }
}

constexpr int kNW = 3, kND = 2;  // noise and accumulation warps per CTA

template <typename S>
size_t sweep2_smem(int tile_slot, int max_parts) {
    constexpr int ESZ = sizeof(S);
    // stage slots are sized for R = 4 (the largest id section)
    const size_t stage = (size_t)NSTG * stage_slot_bytes<ESZ>(max_parts, 4);
    const size_t nbars = NTILE + 2 * NGBUF + 2 * NSTG + 2 * NQ;
    return (size_t)ValueArea<ESZ>::BYTES + (size_t)NTILE * tile_slot + NQ * 32 * 8 + stage + nbars * 8;
}

template <typename S, int C, int R>
static cudaError_t launch2(const Sweep2Params<S> &p, cudaStream_t st) {
    const size_t smem = sweep2_smem<S>(p.tile_slot, p.max_items);
    auto kern = sweep2_kernel<S, C, R, kNW, kND>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<p.ld / C, 32 * (2 + kNW + kND), smem, st>>>(p);
    return cudaGetLastError();
}

template <typename S>
cudaError_t launch_sweep2(const Sweep2Params<S> &p, int C, cudaStream_t st) {
    switch (C) {
        case 8: return launch2<S, 8, 4>(p, st);
        case 16: return launch2<S, 16, 2>(p, st);
        default: return launch2<S, 32, 1>(p, st);
    }
}

template cudaError_t launch_sweep2<double>(const Sweep2Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep2<cd>(const Sweep2Params<cd> &, int, cudaStream_t);
template size_t sweep2_smem<double>(int, int);
template size_t sweep2_smem<cd>(int, int);

}  // namespace mcinv
