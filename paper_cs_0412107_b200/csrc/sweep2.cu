// sweep2.cu -- K1/K2 v2: the CC sweep kernel on a dependency-respecting step
// schedule (plan.h), one warp per CTA.
//
// Lanes = C chains x R row slots (C * R = 32). A step updates up to R rows of
// the warp's C chains at once; the planner guarantees that the rows of a step
// do not depend on each other and that every operand is exactly the one the
// sequential sweep (Eq. 4/5) would read, so z and w are
// bit-identical to the row-by-row order (checked against the oracle).
//
// Per step T the warp
//   1. issues the TMA bulk copy of the record tile of step T+15 (cols,
//      coefficients, smem source offsets, accumulation items) into a 16-slot
//      smem ring (mbarrier complete_tx),
//   2. issues cp.async gathers of the z/w pairs of step T+7's far entries
//      (produced >= 8 steps ago) from the [n][ld] state in HBM into smem,
//   3. runs the serial fma chains of step T reading operands from smem (far
//      entries: the gather buffer; near entries: a ring of the last 8 steps'
//      results), draws phi (Philox4x32-10 + Box-Muller, noise.cuh), writes
//      z_i, w_i to HBM and to the ring,
//   4. in sampling sweeps accumulates diag / pattern via an smem transpose
//      reduction over the chains of an SE group, and the trace w^dagger Q z in
//      registers (Eq. 1/C, Eq. tr).
#include "mcinv_internal.cuh"
#include "noise.cuh"
#include "plan.h"
#include "scalar.cuh"

namespace mcinv {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
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
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <typename S>
__device__ __forceinline__ S lds_s(const unsigned char *p) {
    return *reinterpret_cast<const S *>(p);
}

}  // namespace

template <typename S, int C, int R>
__global__ void __launch_bounds__(32) sweep2_kernel(const Sweep2Params<S> p) {
    constexpr int ESZ = sizeof(S);
    constexpr int ZWSZ = 2 * ESZ;
    constexpr int BLK = 32 * ZWSZ;
    constexpr int GB_OFF = NRING * BLK;
    constexpr int ZERO_OFF = GB_OFF + NRING * KCAP * BLK;
    constexpr int VAL_BYTES = ZERO_OFF + BLK;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *vals = smem;
    unsigned char *tiles = smem + VAL_BYTES;
    unsigned char *stage = tiles + NTILE * p.tile_slot;
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage + (size_t)p.max_items * 32 * ESZ);

    const int lane = threadIdx.x;
    const int c = lane % C, r = lane / C;
    const int cb = blockIdx.x * C;        // first local chain of this CTA
    const int chain = cb + c;             // local chain (< ld)
    const bool active = chain < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);
    const int coff = c * ZWSZ;            // lane's chain offset inside a block row
    const int64_t T0 = (int64_t)p.s_begin * p.steps, T_end = (int64_t)p.s_end * p.steps;
    const int S_n = p.steps;

    // ---- init: barriers, zero block
    for (int b = lane; b < BLK / 16; b += 32) reinterpret_cast<double2 *>(vals + ZERO_OFF)[b] = make_double2(0.0, 0.0);
    if (lane == 0) {
        for (int s = 0; s < NTILE; ++s) mbar_init(smem_u32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    auto issue_tile = [&](int64_t T, int64_t goff, int bytes) {
        if (lane == 0) {
            const int s = (int)(T % NTILE);
            tma_load_1d(smem_u32(tiles + s * p.tile_slot), p.tiles + goff, (uint32_t)bytes, smem_u32(&bars[s]));
        }
    };
    auto wait_tile = [&](int64_t T) {
        mbar_wait(smem_u32(&bars[T % NTILE]), (uint32_t)(((T - T0) / NTILE) & 1));
    };
    auto tile_of = [&](int64_t T) { return tiles + (T % NTILE) * p.tile_slot; };
    // gathers of the far entries of step T (tile already landed)
    auto gather = [&](int64_t T) {
        const unsigned char *tl = tile_of(T);
        const int K = reinterpret_cast<const int *>(tl)[0];
        const TileLayout L{K, 0, R, ESZ};
        for (int k = 0; k < K; ++k) {
            const int2 m = *reinterpret_cast<const int2 *>(tl + L.meta() + 8 * (k * R + r));
            if (m.y >= 0) {
                const unsigned char *src = reinterpret_cast<const unsigned char *>(p.zw + (int64_t)m.y * p.ld + chain);
                const uint32_t dst = smem_u32(vals + m.x + coff);
#pragma unroll
                for (int h = 0; h < ZWSZ / 16; ++h) cp_async16(dst + 16 * h, src + 16 * h);
            }
        }
    };

    // ---- prologue: tiles T0 .. T0+14, ring of the 7 steps before T0, gathers T0 .. T0+6
    for (int64_t T = T0; T < T0 + NTILE - 1 && T < T_end; ++T) {
        const int t = (int)(T % S_n);
        issue_tile(T, p.tile_off[t], (int)(p.tile_off[t + 1] - p.tile_off[t]));
    }
    for (int q = 1; q <= PDIST; ++q) {
        const int64_t T = T0 - q;
        const int t = (int)(((T % S_n) + S_n) % S_n);
        const unsigned char *g = p.tiles + p.tile_off[t];
        const int row = reinterpret_cast<const int *>(g + 32)[r];
        const int flg = reinterpret_cast<const int *>(g + 32)[R + r];
        if (row >= 0 && (flg & 2)) {
            const ZW<S> v = p.zw[(int64_t)row * p.ld + chain];
            *reinterpret_cast<ZW<S> *>(vals + (((T % NRING) + NRING) % NRING) * BLK + r * C * ZWSZ + coff) = v;
        }
    }
    for (int64_t T = T0; T < T0 + PDIST; ++T) {
        if (T < T_end) {
            wait_tile(T);
            gather(T);
        }
        cp_async_commit();
    }
    __syncwarp();

    S acc_z = zero_s<S>(), acc_w = zero_s<S>(), tr = zero_s<S>();
    const bool want_tr = (p.outputs & OUT_TRACE) != 0;
    for (int64_t T = T0; T < T_end; ++T) {
        const unsigned char *tl = tile_of(T);
        const int *hdr = reinterpret_cast<const int *>(tl);
        const int K = hdr[0], I = hdr[1];
        // 1. record tile of step T+15 into the slot of step T-1
        if (T + NTILE - 1 < T_end) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_tile(T + NTILE - 1, *reinterpret_cast<const int64_t *>(tl + 16), hdr[2]);
        }
        // 2. gathers for step T+7 (its far entries were produced at steps <= T-1)
        if (T + PDIST < T_end) {
            wait_tile(T + PDIST);
            gather(T + PDIST);
        }
        cp_async_commit();
        // 3. operands of step T have landed
        cp_async_wait<PDIST>();

        const TileLayout L{K, I, R, ESZ};
        const int flags = reinterpret_cast<const int *>(tl + 32)[R + r];
        if (flags & 1) {
            acc_z = zero_s<S>();
            acc_w = zero_s<S>();
        }
        for (int k = 0; k < K; ++k) {
            const int off = reinterpret_cast<const int *>(tl + L.meta())[2 * (k * R + r)];
            const S a = lds_s<S>(tl + L.coef() + 2 * ESZ * (k * R + r));
            const S b = lds_s<S>(tl + L.coef() + 2 * ESZ * (k * R + r) + ESZ);
            const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vals + off + coff);
            acc_z = fma_s(a, v.z, acc_z);
            acc_w = fma_s(b, v.w, acc_w);
        }
        const bool last = (flags & 2) != 0;
        const int64_t s_loc = T / S_n;  // local sweep index of this launch's sweep range
        const bool sampling = s_loc >= p.burn_in;
        S zi = zero_s<S>(), wi = zero_s<S>();
        if (last) {
            const int row = reinterpret_cast<const int *>(tl + 32)[r];
            double phi;
            if (p.noise == 0)
                phi = gaussian(static_cast<uint32_t>(row), p.sweep_abs0 + static_cast<uint32_t>(s_loc), gchain, p.key0,
                               p.key1);
            else
                phi = p.noise == 2 ? 1.0 : 0.0;
            const S dl = lds_s<S>(tl + L.dsig() + r * ESZ);
            const S sg = lds_s<S>(tl + L.dsig() + (R + r) * ESZ);
            zi = fma_s(neg_s(dl), acc_z, scale_s(sg, phi));
            wi = fma_s(neg_s(conj_s(dl)), acc_w, scale_s(conj_s(sg), phi));
            p.zw[(int64_t)row * p.ld + chain] = ZW<S>{zi, wi};
            *reinterpret_cast<ZW<S> *>(vals + (T % NRING) * BLK + r * C * ZWSZ + coff) = ZW<S>{zi, wi};
            if ((p.outputs & OUT_FULL) && sampling) {
                const int64_t t = s_loc - p.snap_s0;
                p.snap_x[(t * p.n + row) * p.ld + chain] = zi;
                p.snap_y[(t * p.n + row) * p.ld + chain] = wi;
            }
        }
        if (sampling && I > 0) {
            // 4. items: products (staged for the group reduction) and trace registers
            S qz = zero_s<S>(), qw = zero_s<S>();
            const bool live = last && active;
            for (int q = 0; q < I; ++q) {
                const unsigned char *it = tl + L.items() + L.item_bytes() * (q * R + r);
                const int4 w4 = *reinterpret_cast<const int4 *>(it);
                const int op = w4.x & 7;
                ZW<S> pv{zero_s<S>(), zero_s<S>()};
                if (op == IT_PAT_ZI || op == IT_PAT_ZO || op == IT_QROW || op == IT_QCOL) {
                    if (w4.x & 8) pv = *reinterpret_cast<const ZW<S> *>(vals + w4.w + coff);
                    else if (live) pv = p.zw[(int64_t)w4.z * p.ld + chain];
                }
                S prod = zero_s<S>();
                switch (op) {
                    case IT_DIAG:
                    case IT_PAT_SELF: prod = zwc_s(zi, wi); break;
                    case IT_PAT_ZI: prod = zwc_s(zi, pv.w); break;
                    case IT_PAT_ZO: prod = zwc_s(pv.z, wi); break;
                    case IT_QROW: qz = add_s(qz, mul_s(lds_s<S>(it + 16), pv.z)); break;
                    case IT_QROW_SELF: qz = add_s(qz, mul_s(lds_s<S>(it + 16), zi)); break;
                    case IT_QCOL: qw = add_s(qw, mul_s(lds_s<S>(it + 16), conj_s(pv.w))); break;
                    default: break;
                }
                *reinterpret_cast<S *>(stage + (q * 32 + lane) * ESZ) = live ? prod : zero_s<S>();
            }
            if (want_tr && live) tr = add_s(tr, add_s(zwc_s(qz, wi), mul_s(zi, qw)));
            __syncwarp();
            // group sums: one task per (item, row slot, SE group); groups wider
            // than the CTA's C chains are completed with atomics across CTAs
            const int gse = p.gs < C ? p.gs : C;
            const int gpr = C / gse;  // groups (or group parts) per row slot
            const int ntask = I * R * gpr;
            for (int tk = lane; tk < ntask; tk += 32) {
                const int q = tk / (R * gpr), rem = tk % (R * gpr);
                const int r2 = rem / gpr, g2 = rem % gpr;
                const unsigned char *it = tl + L.items() + L.item_bytes() * (q * R + r2);
                const int2 w2 = *reinterpret_cast<const int2 *>(it);
                const int op = w2.x & 7;
                if (op < IT_DIAG || op > IT_PAT_SELF) continue;
                const int c0 = g2 * gse;
                if (cb + c0 >= p.chains) continue;
                S sum = zero_s<S>();
                for (int cc = 0; cc < gse; ++cc)
                    sum = add_s(sum, *reinterpret_cast<const S *>(stage + (q * 32 + r2 * C + c0 + cc) * ESZ));
                const int64_t grp = (cb + c0) / p.gs;
                double *dst = op == IT_DIAG ? p.slot_diag + (grp * p.n + w2.y) * (ESZ / 8)
                                            : p.slot_pat + (grp * p.pcount + w2.y) * (ESZ / 8);
                if (p.gs > C) atomic_add_to(dst, sum);
                else add_to(dst, sum);
            }
        }
        __syncwarp();
    }
    // trace: sum the lane registers over row slots and the chains of each group
    if (want_tr) {
        __syncwarp();
        *reinterpret_cast<S *>(stage + lane * ESZ) = active ? tr : zero_s<S>();
        __syncwarp();
        const int gse = p.gs < C ? p.gs : C;
        const int ngrp = C / gse;
        if (lane < ngrp && cb + lane * gse < p.chains) {
            S sum = zero_s<S>();
            for (int r2 = 0; r2 < R; ++r2)
                for (int cc = 0; cc < gse; ++cc)
                    sum = add_s(sum, *reinterpret_cast<const S *>(stage + (r2 * C + lane * gse + cc) * ESZ));
            double *dst = p.slot_trace + (int64_t)((cb + lane * gse) / p.gs) * (ESZ / 8);
            if (p.gs > C) atomic_add_to(dst, sum);
            else add_to(dst, sum);
        }
    }
}

template <typename S>
size_t sweep2_smem(int tile_slot, int max_items) {
    constexpr int BLK = 32 * 2 * sizeof(S);
    const size_t vals = (size_t)(NRING + NRING * KCAP + 1) * BLK;
    const int mi = max_items > 1 ? max_items : 1;
    return vals + (size_t)NTILE * tile_slot + (size_t)mi * 32 * sizeof(S) + NTILE * 8;
}

template <typename S, int C, int R>
static cudaError_t launch2(const Sweep2Params<S> &p, cudaStream_t st) {
    const size_t smem = sweep2_smem<S>(p.tile_slot, p.max_items);
    cudaError_t e = cudaFuncSetAttribute(sweep2_kernel<S, C, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int blocks = p.ld / C;
    sweep2_kernel<S, C, R><<<blocks, 32, smem, st>>>(p);
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
