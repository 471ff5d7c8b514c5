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
//                 result ring, FULL-output snapshots, D's records, trace.
//   B  (1 warp)   producer: TMA bulk copy of the record tile of step U+8
//                 (cols, coefficients, smem source offsets, accumulation
//                 records) and cp.async gathers of step U's far operands
//                 (>= 8 steps old) from the [n][ld] state in HBM; waits for
//                 A(U-8) and, for gather-slot reuse, D(U-NGB+1).
//   D  (ND warps) accumulation (sampling sweeps): A hands each finished row's
//                 accumulation records (value offsets, slots) to D through a
//                 record ring; D forms the diag and pattern products (Eq. 1/C,
//                 P:173-176) from the values in smem, sums them over the
//                 chains of an SE group and does one RMW (or RED) per group
//                 slot. Deep gather/result buffers (16/32 steps for f64) let
//                 D lag A. The trace w^dagger Q z (Eq. tr) is
//                 summed in A's registers.
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
// Protocol watchdog: a wait that does not complete in 20 s records who waited
// (block, warp, barrier, parity, step) in g_sweep2_dbg, raises g_sweep2_abort
// so that every other wait returns, and the kernel drains; the host reports
// it as a divergence-style failure (mcinv_result) with the record on stderr.
__device__ unsigned int g_sweep2_abort;
__device__ unsigned int g_sweep2_dbg[8];
__device__ unsigned int g_sweep2_warps[8][4];  // block dbg[0]: per warp {bar, parity, tag, 1}

// suspend-hinted try_wait: the thread sleeps (up to ~1 us) instead of spinning
__device__ __forceinline__ uint32_t mbar_try_sleep(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000u)
        : "memory");
    return ok;
}

__device__ __noinline__ void mbar_wait_slow(uint32_t bar, uint32_t parity, uint32_t tag) {
    const uint64_t t0 = globaltimer_ns();
    for (uint32_t it = 1;; ++it) {
        if (mbar_try_sleep(bar, parity)) return;
        if ((it & 255) != 0) continue;
        if (*reinterpret_cast<volatile unsigned int *>(&g_sweep2_abort)) {
            if (blockIdx.x == *reinterpret_cast<volatile unsigned int *>(&g_sweep2_dbg[0]) &&
                (threadIdx.x & 31) == 0) {
                const int w = (threadIdx.x >> 5) & 7;
                g_sweep2_warps[w][0] = bar;
                g_sweep2_warps[w][1] = parity;
                g_sweep2_warps[w][2] = tag;
                g_sweep2_warps[w][3] = 1;
            }
            return;
        }
        if (globaltimer_ns() - t0 > 20000000000ull) {
            if (atomicCAS(&g_sweep2_abort, 0u, 1u) == 0u) {
                g_sweep2_dbg[0] = blockIdx.x;
                g_sweep2_dbg[1] = threadIdx.x >> 5;
                g_sweep2_dbg[2] = bar;
                g_sweep2_dbg[3] = parity;
                g_sweep2_dbg[4] = tag;
                __threadfence();
            }
            return;
        }
    }
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, uint32_t tag = 0) {
    if (mbar_try(bar, parity)) return;
    mbar_wait_slow(bar, parity, tag);
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

// Record-ring slot (A -> D), one per step: int P (header, 16 B), then
// int4 rec[P+1][R]: {smem value offset, pzi, pzo, -} per partner record and,
// at index P, {offset of the row's own z_i, w_i in the ring, dslot, pslot, -};
// slots are -1 for row slots whose row did not finish in the step.
__host__ __device__ inline int rec_slot_bytes(int max_parts, int R) { return 16 + 16 * (max_parts + 1) * R; }
// D scratch: products [2 (P+1)][32] for the transpose reduction
template <int ESZ>
__host__ __device__ inline int dstage_bytes(int max_parts) { return 2 * (max_parts + 1) * 32 * ESZ; }

// The serial part of Eq. (4)/(5) for one step: load all KU operands first
// (entries k >= K read the zero block with coefficient 0, an exact no-op), then
// the two fma chains in ascending CSR order (reading R10).
template <typename S, int KU, int R>
__device__ __forceinline__ void fma_chain(int K, const int2 *meta, const unsigned char *cf,
                                          const unsigned char *vlane, const unsigned char *zero, S &acc_z,
                                          S &acc_w) {
    constexpr int ESZ = sizeof(S);
    ZW<S> v[KU];
    S a[KU], b[KU];
#pragma unroll
    for (int k = 0; k < KU; ++k) {
        const bool in = k < K;
        const unsigned char *src = in ? vlane + meta[k * R].x : zero;
        v[k] = *reinterpret_cast<const ZW<S> *>(src);
        a[k] = in ? *reinterpret_cast<const S *>(cf + 2 * ESZ * R * k) : zero_s<S>();
        b[k] = in ? *reinterpret_cast<const S *>(cf + 2 * ESZ * R * k + ESZ) : zero_s<S>();
    }
#pragma unroll
    for (int k = 0; k < KU; ++k) {
        acc_z = fma_s(a[k], v[k].z, acc_z);
        acc_w = fma_s(b[k], v[k].w, acc_w);
    }
}

// Warp roles: 0 = A; 1..NW = N; NW+1 = B; NW+2 .. NW+1+ND = D. Warps share an
// SMSP by index mod 4, so A pairs with B and each D with a noise warp.
template <typename S, int C, int R, int NW, int ND>
__global__ void __launch_bounds__(32 * (2 + NW + ND)) sweep2_kernel(const Sweep2Params<S> p) {
    constexpr int ESZ = sizeof(S);
    constexpr int ZWSZ = 2 * ESZ;
    using VA = ValueArea<ESZ>;
    constexpr int BLK = VA::BLK;
    constexpr int NGB = VA::NGB, NRG = VA::NRG;
    constexpr int WB = NW + 1;  // producer warp

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *vals = smem;
    unsigned char *tiles = smem + VA::BYTES;
    double *noise = reinterpret_cast<double *>(tiles + NTILE * p.tile_slot);   // [NQ][32]
    unsigned char *recring = reinterpret_cast<unsigned char *>(noise + NQ * 32);  // [NGB] record slots
    const int rec_bytes = rec_slot_bytes(p.max_items, R);
    unsigned char *dstage0 = recring + (size_t)NGB * rec_bytes;
    const int dst_bytes = dstage_bytes<ESZ>(p.max_items);
    uint64_t *bars = reinterpret_cast<uint64_t *>(dstage0 + (size_t)ND * dst_bytes);
    const uint32_t b_tile = smem_u32(bars);               // [NTILE] TMA complete_tx
    if (threadIdx.x == 0 && blockIdx.x == 0) g_sweep2_dbg[5] = b_tile;
    const uint32_t b_gather = b_tile + 8 * NTILE;         // [NGB] 32 cp.async arrivals
    const uint32_t b_adone = b_gather + 8 * NGB;          // [NGB] A finished step
    const uint32_t b_ddone = b_adone + 8 * NGB;           // [NGB] D finished (sampling) step
    const uint32_t b_nfull = b_ddone + 8 * NGB;           // [NQ] noise ready
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
    // first sampling step: D and the d_done barriers count their phases from here
    const uint32_t Ts = min(T_end, max(T0, (uint32_t)p.burn_in * S_n));
    const uint32_t tile_slot = (uint32_t)p.tile_slot;
    const bool want_tr = (p.outputs & OUT_TRACE) != 0;
    const bool want_red = (p.outputs & (OUT_DIAG | OUT_PATTERN)) != 0;
    auto tile_of = [&](uint32_t T) { return tiles + (T % NTILE) * tile_slot; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NTILE; ++s) mbar_init(b_tile + 8 * s, 1);
        for (int s = 0; s < NGB; ++s) {
            mbar_init(b_gather + 8 * s, 32);
            mbar_init(b_adone + 8 * s, 1);
            mbar_init(b_ddone + 8 * s, ND > 0 ? 1 : 1);
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
                *reinterpret_cast<ZW<S> *>(vals + (((T % NRG) + NRG) % NRG) * BLK + roff + coff) =
                    p.zw[(int64_t)row * p.ld + chain];
        }
    }
    __syncthreads();

    if (warp == WB) {
        // ================= B: tiles and gathers
        const unsigned char *zw_chain = reinterpret_cast<const unsigned char *>(p.zw + chain);
        const int64_t row_bytes = (int64_t)p.ld * ZWSZ;
        const unsigned char *gtiles = p.tiles;
        const uint32_t vbase = smem_u32(vals) + coff;
        const bool wait_d = want_red;  // D reads gather slots of steps T and T-1
        if (lane == 0)
            for (uint32_t T = T0; T < T0 + 8 && T < T_end; ++T) {
                const int t = (int)(T % S_n);
                tma_load_1d(smem_u32(tile_of(T)), gtiles + p.tile_off[t], (uint32_t)(p.tile_off[t + 1] - p.tile_off[t]),
                            b_tile + 8 * (T % NTILE));
            }
        for (uint32_t U = T0; U < T_end; ++U) {
            // far operands of step U were produced at steps <= U-8 (A done); the
            // gather slot U % NGB was last read by A(U-NGB) and by D(U-NGB), D(U-NGB+1)
            if (U >= T0 + 8) mbar_wait(b_adone + 8 * ((U - 8) % NGB), par<NGB>(U - 8, T0), U);
            if (wait_d && U + 1 >= Ts + NGB) mbar_wait(b_ddone + 8 * ((U + 1 - NGB) % NGB), par<NGB>(U + 1 - NGB, Ts), U);
            mbar_wait(b_tile + 8 * (U % NTILE), par<NTILE>(U, T0), U);
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
            cp_async_arrive(b_gather + 8 * (U % NGB));
        }
    } else if (warp == 0) {
        // ================= A: the serial fma chains
        S acc_z = zero_s<S>(), acc_w = zero_s<S>(), tr = zero_s<S>();
        ZW<S> *zw_chain = p.zw + chain;
        const unsigned char *vlane = vals + coff;
        unsigned char *ring_lane = vals + roff + coff;
        uint32_t ok_g = 0, ok_n = 0;
        for (uint32_t T = T0; T < T_end; ++T) {
            if (!ok_g) mbar_wait(b_gather + 8 * (T % NGB), par<NGB>(T, T0), T);
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
            if (K <= 4) fma_chain<S, 4, R>(K, meta, cf, vlane, vals + VA::ZERO, acc_z, acc_w);
            else fma_chain<S, KCAP, R>(K, meta, cf, vlane, vals + VA::ZERO, acc_z, acc_w);
            // probe the next step's gathers while the fma chains drain
            const uint32_t Tn = T + 1;
            ok_g = Tn < T_end ? mbar_test(b_gather + 8 * (Tn % NGB), par<NGB>(Tn, T0)) : 1u;
            if (!ok_n) mbar_wait(b_nfull + 8 * (T % NQ), par<NQ>(T, T0), T);
            const bool last = (flags & 2) != 0;
            const bool sampling = T >= Ts;
            S zi = zero_s<S>(), wi = zero_s<S>();
            if (last) {
                const int row = reinterpret_cast<const int *>(tl + 32)[r];
                const double phi = noise[(T % NQ) * 32 + lane];
                const S dl = lds_s<S>(tl + L.dsq() + r * ESZ);
                const S sg = lds_s<S>(tl + L.dsq() + (R + r) * ESZ);
                zi = fma_s(neg_s(dl), acc_z, scale_s(sg, phi));
                wi = fma_s(neg_s(conj_s(dl)), acc_w, scale_s(conj_s(sg), phi));
                zw_chain[(int64_t)row * p.ld] = ZW<S>{zi, wi};
                *reinterpret_cast<ZW<S> *>(ring_lane + (T % NRG) * BLK) = ZW<S>{zi, wi};
                if ((p.outputs & OUT_FULL) && sampling) {
                    const int64_t t = (int64_t)(T / S_n) - p.snap_s0;
                    p.snap_x[(t * p.n + row) * p.ld + chain] = zi;
                    p.snap_y[(t * p.n + row) * p.ld + chain] = wi;
                }
            }
            ok_n = Tn < T_end ? mbar_test(b_nfull + 8 * (Tn % NQ), par<NQ>(Tn, T0)) : 1u;
            if (sampling && (want_red || want_tr)) {
                const unsigned char *pr = tl + L.part() + L.part_bytes() * r;
                if (want_red && c == 0) {
                    // hand the row's accumulation records to D (one lane per row slot)
                    unsigned char *rs_ = recring + (T % NGB) * rec_bytes;
                    int4 *rec = reinterpret_cast<int4 *>(rs_ + 16) + r;
                    for (int q = 0; q < P; ++q) {
                        int4 v = *reinterpret_cast<const int4 *>(pr + q * L.part_bytes() * R);
                        if (!last) v.y = v.z = -1;
                        rec[q * R] = v;
                    }
                    const int *rs = reinterpret_cast<const int *>(tl + 32);
                    rec[P * R] = last ? make_int4((int)((T % NRG) * BLK) + roff, rs[2 * R + r], rs[3 * R + r], 0)
                                      : make_int4(0, -1, -1, 0);
                    if (r == 0) reinterpret_cast<int *>(rs_)[0] = P;
                }
                if (want_tr && last) {
                    S qz = mul_s(lds_s<S>(tl + L.dsq() + (2 * R + r) * ESZ), zi);
                    S qw = zero_s<S>();
                    for (int q = 0; q < P; ++q) {
                        const unsigned char *pq = pr + q * L.part_bytes() * R;
                        const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vlane + reinterpret_cast<const int *>(pq)[0]);
                        qz = add_s(qz, mul_s(lds_s<S>(pq + 16), v.z));
                        qw = add_s(qw, mul_s(lds_s<S>(pq + 16 + ESZ), conj_s(v.w)));
                    }
                    if (active) tr = add_s(tr, add_s(zwc_s(qz, wi), mul_s(zi, qw)));
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(b_nempty + 8 * (T % NQ));
                mbar_arrive(b_adone + 8 * (T % NGB));
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
        // ================= D: diag / pattern products and group reductions,
        // sampling steps Ts + dw, Ts + dw + ND, ...; reads values in place
        if (want_red) {
            const int dw = warp - WB - 1;
            S *st = reinterpret_cast<S *>(dstage0 + (size_t)dw * dst_bytes);
            const int gse = p.gs < C ? p.gs : C;
            const int lg_gse = __ffs(gse) - 1;
            const int lg_tpr = 5 - lg_gse;          // tasks per product record: 32 / gse
            const int lg_gpr = __ffs(C / gse) - 1;  // group parts per row slot
            const bool use_atomic = p.gs > C || ND > 1;
            const unsigned char *vlane = vals + coff;
            // every step is waited in order (also in burn-in): a parity wait may
            // only target the phase right after the last one observed
            for (uint32_t T = T0 + dw; T < T_end; T += ND) {
                mbar_wait(b_adone + 8 * (T % NGB), par<NGB>(T, T0), T);
                if (T < Ts) continue;
                const unsigned char *rs_ = recring + (T % NGB) * rec_bytes;
                const int P = reinterpret_cast<const int *>(rs_)[0];
                const int4 *rec = reinterpret_cast<const int4 *>(rs_ + 16);
                const int4 self = rec[P * R + r];
                const ZW<S> me = *reinterpret_cast<const ZW<S> *>(vlane + self.x);
                const bool live = self.y >= 0 || self.z >= 0;
                const S sp = (live && active) ? zwc_s(me.z, me.w) : zero_s<S>();
                st[(2 * P) * 32 + lane] = sp;       // diag
                st[(2 * P + 1) * 32 + lane] = sp;   // pattern (i,i)
                for (int q = 0; q < P; ++q) {
                    const int4 rc = rec[q * R + r];
                    const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vlane + rc.x);
                    st[(2 * q) * 32 + lane] = zwc_s(me.z, v.w);
                    st[(2 * q + 1) * 32 + lane] = zwc_s(v.z, me.w);
                }
                __syncwarp();
                // task = (product record qh, row slot r2, group part g2): sum gse chains, one RMW/RED
                const int nt = (2 * P + 2) << lg_tpr;
                for (int tk = lane; tk < nt; tk += 32) {
                    const int qh = tk >> lg_tpr, rem = tk & ((1 << lg_tpr) - 1);
                    const int r2 = rem >> lg_gpr, g2 = rem & ((1 << lg_gpr) - 1);
                    const int4 rc = rec[(qh >> 1) * R + r2];
                    const int slot = (qh & 1) ? rc.z : rc.y;
                    const int c0 = g2 << lg_gse;
                    if (slot < 0 || cb + c0 >= p.chains) continue;
                    const S *sv = st + qh * 32 + r2 * C + c0;
                    S sum = sv[0];
                    for (int cc = 1; cc < gse; ++cc) sum = add_s(sum, sv[cc]);
                    const bool to_diag = qh == 2 * P;
                    const int64_t grp = (cb + c0) / p.gs;
                    double *dst = to_diag ? p.slot_diag + (grp * p.n + slot) * (ESZ / 8)
                                          : p.slot_pat + (grp * p.pcount + slot) * (ESZ / 8);
                    if (use_atomic) atomic_add_to(dst, sum);
                    else add_to(dst, sum);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(b_ddone + 8 * (T % NGB));
            }
        }
    } else {
        // ================= N: noise, steps T0 + w, T0 + w + NW, ...
        const int w = warp - 1;
        for (uint32_t T = T0 + w; T < T_end; T += NW) {
            if (T >= T0 + NQ) mbar_wait(b_nempty + 8 * (T % NQ), par<NQ>(T - NQ, T0), T);
            mbar_wait(b_tile + 8 * (T % NTILE), par<NTILE>(T, T0), T);
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
    using VA = ValueArea<ESZ>;
    // record slots are sized for R = 4 (the largest)
    const size_t recs = (size_t)VA::NGB * rec_slot_bytes(max_parts, 4);
    const size_t dst = (size_t)kND * dstage_bytes<ESZ>(max_parts);
    const size_t nbars = NTILE + 3 * VA::NGB + 2 * NQ;
    return (size_t)VA::BYTES + (size_t)NTILE * tile_slot + NQ * 32 * 8 + recs + dst + nbars * 8;
}

template <typename S, int C, int R>
static cudaError_t launch2(const Sweep2Params<S> &p, cudaStream_t st) {
    const size_t smem = sweep2_smem<S>(p.tile_slot, p.max_items);
    auto kern = sweep2_kernel<S, C, R, kNW, kND>;
    static const unsigned int zeros[32] = {0};
    cudaMemcpyToSymbolAsync(g_sweep2_abort, zeros, sizeof(unsigned int), 0, cudaMemcpyHostToDevice, st);
    cudaMemcpyToSymbolAsync(g_sweep2_warps, zeros, sizeof(zeros), 0, cudaMemcpyHostToDevice, st);
    cudaMemcpyToSymbolAsync(g_sweep2_dbg, zeros, 8 * sizeof(unsigned int), 0, cudaMemcpyHostToDevice, st);
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

// 1 if a protocol watchdog fired since the last launch; dbg[6] receives the record
int sweep2_debug(unsigned int *dbg) {
    unsigned int a = 0;
    cudaMemcpyFromSymbol(&a, g_sweep2_abort, sizeof(a));
    if (dbg) {
        cudaMemcpyFromSymbol(dbg, g_sweep2_dbg, 6 * sizeof(unsigned int));
        cudaMemcpyFromSymbol(dbg + 6, g_sweep2_warps, 32 * sizeof(unsigned int));
    }
    return (int)a;
}

template cudaError_t launch_sweep2<double>(const Sweep2Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep2<cd>(const Sweep2Params<cd> &, int, cudaStream_t);
template size_t sweep2_smem<double>(int, int);
template size_t sweep2_smem<cd>(int, int);

}  // namespace mcinv
