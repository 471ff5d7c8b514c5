// sweep2.cu -- K1/K2 (v2): the CC sweep on a dependency-respecting step
// schedule (plan.h), warp-specialized.
//
// One CTA owns C chains; lanes = C chains x R row slots (C * R = 32). The
// planner guarantees that the rows of a step do not depend on each other and
// that every operand is exactly the one the sequential sweep (Eq. 4/5,
// PAPER.md:157-160) reads, so z and w are bit-identical to row-by-row order.
//
// Warp roles (all synchronised with mbarriers, per step slot):
//   A  (warp 0)   the serial part only: for each step, the fma chains of
//                 Eq. (4)/(5) over smem operands, z_i, w_i to HBM and to the
//                 16-step result ring, FULL-output snapshots.
//   B  (warp 1)   producer: TMA bulk copy of the record tile of step U+8
//                 (cols, coefficients, smem source offsets, accumulation
//                 records) and cp.async gathers of step U's far operands
//                 (>= 8 steps old) from the [n][ld] state in HBM.
//   D  (warp 2)   accumulation (sampling sweeps): diag, pattern and trace
//                 products of the rows finished in the step (Eq. 1/C, Eq. tr,
//                 P:173-182), smem transpose-reduction over the chains of an
//                 SE group, one RMW (or RED) per group slot.
//   N  (warps 3+) noise: phi(row, sweep, chain) by Philox4x32-10 + Box-Muller
//                 (noise.cuh) into an smem ring, NW warps round-robin.
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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
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

// phase parity of the use of a step-indexed barrier slot (T relative to T0)
__device__ __forceinline__ uint32_t par(int64_t T, int64_t T0, int nslots) {
    return (uint32_t)(((T - T0) / nslots) & 1);
}

}  // namespace

template <typename S, int C, int R, int NW>
__global__ void __launch_bounds__(32 * (3 + NW)) sweep2_kernel(const Sweep2Params<S> p) {
    constexpr int ESZ = sizeof(S);
    constexpr int ZWSZ = 2 * ESZ;
    using VA = ValueArea<ESZ>;
    constexpr int BLK = VA::BLK;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *vals = smem;
    unsigned char *tiles = smem + VA::BYTES;
    double *noise = reinterpret_cast<double *>(tiles + NTILE * p.tile_slot);   // [NQ][32]
    unsigned char *stage = reinterpret_cast<unsigned char *>(noise + NQ * 32);  // D products [2P+2][32]
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage + (size_t)(2 * p.max_items + 2) * 32 * ESZ);
    uint64_t *b_tile = bars;                   // [NTILE] TMA complete_tx
    uint64_t *b_gather = b_tile + NTILE;       // [NGBUF] 32 cp.async arrivals
    uint64_t *b_adone = b_gather + NGBUF;      // [NGBUF] A finished step
    uint64_t *b_ddone = b_adone + NGBUF;       // [NGBUF] D finished step
    uint64_t *b_nfull = b_ddone + NGBUF;       // [NQ] noise ready
    uint64_t *b_nempty = b_nfull + NQ;         // [NQ] noise consumed

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = lane % C, r = lane / C;
    const int cb = blockIdx.x * C;
    const int chain = cb + c;
    const bool active = chain < p.chains;
    const uint32_t gchain = p.chain0 + static_cast<uint32_t>(chain);
    const int coff = c * ZWSZ;
    const int roff = r * C * ZWSZ;
    const int64_t T0 = (int64_t)p.s_begin * p.steps, T_end = (int64_t)p.s_end * p.steps;
    const int S_n = p.steps;
    auto tile_of = [&](int64_t T) { return tiles + (T % NTILE) * p.tile_slot; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NTILE; ++s) mbar_init(smem_u32(&b_tile[s]), 1);
        for (int s = 0; s < NGBUF; ++s) {
            mbar_init(smem_u32(&b_gather[s]), 32);
            mbar_init(smem_u32(&b_adone[s]), 1);
            mbar_init(smem_u32(&b_ddone[s]), 1);
        }
        for (int s = 0; s < NQ; ++s) {
            mbar_init(smem_u32(&b_nfull[s]), 1);
            mbar_init(smem_u32(&b_nempty[s]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        // zero block and the ring of the 7 steps before T0 (from the state)
        for (int b = lane; b < BLK / 16; b += 32)
            reinterpret_cast<double2 *>(vals + VA::ZERO)[b] = make_double2(0.0, 0.0);
        for (int q = 1; q <= PDIST; ++q) {
            const int64_t T = T0 - q;
            const int t = (int)(((T % S_n) + S_n) % S_n);
            const int *g = reinterpret_cast<const int *>(p.tiles + p.tile_off[t] + 32);
            const int row = g[r], flg = g[R + r];
            if (row >= 0 && (flg & 2))
                *reinterpret_cast<ZW<S> *>(vals + (((T % NRING) + NRING) % NRING) * BLK + roff + coff) =
                    p.zw[(int64_t)row * p.ld + chain];
        }
    }
    __syncthreads();

    if (warp == 1) {
        // ================= B: tiles and gathers
        if (lane == 0)
            for (int64_t T = T0; T < T0 + 8 && T < T_end; ++T) {
                const int t = (int)(T % S_n);
                tma_load_1d(smem_u32(tile_of(T)), p.tiles + p.tile_off[t], (uint32_t)(p.tile_off[t + 1] - p.tile_off[t]),
                            smem_u32(&b_tile[T % NTILE]));
            }
        for (int64_t U = T0; U < T_end; ++U) {
            if (U - 8 >= T0) mbar_wait(smem_u32(&b_adone[U % NGBUF]), par(U - 8, T0, NGBUF));
            if (U - 7 >= T0) mbar_wait(smem_u32(&b_ddone[(U - 7) % NGBUF]), par(U - 7, T0, NGBUF));
            mbar_wait(smem_u32(&b_tile[U % NTILE]), par(U, T0, NTILE));
            const unsigned char *tl = tile_of(U);
            const int *hdr = reinterpret_cast<const int *>(tl);
            if (lane == 0 && U + 8 < T_end) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_load_1d(smem_u32(tile_of(U + 8)), p.tiles + *reinterpret_cast<const int64_t *>(tl + 16),
                            (uint32_t)hdr[2], smem_u32(&b_tile[(U + 8) % NTILE]));
            }
            const TileLayout L{hdr[0], hdr[1], R, ESZ};
            for (int k = 0; k < L.K; ++k) {
                const int2 m = *reinterpret_cast<const int2 *>(tl + L.meta() + 8 * (k * R + r));
                if (m.y >= 0) {
                    const unsigned char *src =
                        reinterpret_cast<const unsigned char *>(p.zw + (int64_t)m.y * p.ld + chain);
                    const uint32_t dst = smem_u32(vals + m.x + coff);
#pragma unroll
                    for (int h = 0; h < ZWSZ / 16; ++h) cp_async16(dst + 16 * h, src + 16 * h);
                }
            }
            cp_async_arrive(smem_u32(&b_gather[U % NGBUF]));
        }
    } else if (warp == 0) {
        // ================= A: the serial fma chains
        S acc_z = zero_s<S>(), acc_w = zero_s<S>();
        for (int64_t T = T0; T < T_end; ++T) {
            mbar_wait(smem_u32(&b_gather[T % NGBUF]), par(T, T0, NGBUF));
            const unsigned char *tl = tile_of(T);
            const int *hdr = reinterpret_cast<const int *>(tl);
            const TileLayout L{hdr[0], hdr[1], R, ESZ};
            const int flags = reinterpret_cast<const int *>(tl + 32)[R + r];
            if (flags & 1) {
                acc_z = zero_s<S>();
                acc_w = zero_s<S>();
            }
            for (int k = 0; k < L.K; ++k) {
                const int off = reinterpret_cast<const int *>(tl + L.meta())[2 * (k * R + r)];
                const unsigned char *cf = tl + L.coef() + 2 * ESZ * (k * R + r);
                const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vals + off + coff);
                acc_z = fma_s(lds_s<S>(cf), v.z, acc_z);
                acc_w = fma_s(lds_s<S>(cf + ESZ), v.w, acc_w);
            }
            mbar_wait(smem_u32(&b_nfull[T % NQ]), par(T, T0, NQ));
            if (flags & 2) {
                const int row = reinterpret_cast<const int *>(tl + 32)[r];
                const double phi = noise[(T % NQ) * 32 + lane];
                const S dl = lds_s<S>(tl + L.dsq() + r * ESZ);
                const S sg = lds_s<S>(tl + L.dsq() + (R + r) * ESZ);
                const S zi = fma_s(neg_s(dl), acc_z, scale_s(sg, phi));
                const S wi = fma_s(neg_s(conj_s(dl)), acc_w, scale_s(conj_s(sg), phi));
                p.zw[(int64_t)row * p.ld + chain] = ZW<S>{zi, wi};
                *reinterpret_cast<ZW<S> *>(vals + (T % NRING) * BLK + roff + coff) = ZW<S>{zi, wi};
                const int64_t s_loc = T / S_n;
                if ((p.outputs & OUT_FULL) && s_loc >= p.burn_in) {
                    const int64_t t = s_loc - p.snap_s0;
                    p.snap_x[(t * p.n + row) * p.ld + chain] = zi;
                    p.snap_y[(t * p.n + row) * p.ld + chain] = wi;
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&b_nempty[T % NQ]));
                mbar_arrive(smem_u32(&b_adone[T % NGBUF]));
            }
        }
    } else if (warp == 2) {
        // ================= D: accumulation
        const bool want_tr = (p.outputs & OUT_TRACE) != 0;
        const bool want_red = (p.outputs & (OUT_DIAG | OUT_PATTERN)) != 0;
        const int gse = p.gs < C ? p.gs : C;
        const int gpr = C / gse;
        S tr = zero_s<S>();
        S *st = reinterpret_cast<S *>(stage);
        for (int64_t T = T0; T < T_end; ++T) {
            mbar_wait(smem_u32(&b_adone[T % NGBUF]), par(T, T0, NGBUF));
            const int64_t s_loc = T / S_n;
            if (s_loc >= p.burn_in && (want_tr || want_red)) {
                const unsigned char *tl = tile_of(T);
                const int *hdr = reinterpret_cast<const int *>(tl);
                const TileLayout L{hdr[0], hdr[1], R, ESZ};
                const int *rs = reinterpret_cast<const int *>(tl + 32);
                const bool live = (rs[R + r] & 2) && active;
                const ZW<S> me = *reinterpret_cast<const ZW<S> *>(vals + (T % NRING) * BLK + roff + coff);
                const S self = zwc_s(me.z, me.w);
                st[(2 * L.P) * 32 + lane] = live ? self : zero_s<S>();      // diag
                st[(2 * L.P + 1) * 32 + lane] = live ? self : zero_s<S>();  // pattern (i,i)
                S qz = mul_s(lds_s<S>(tl + L.dsq() + (2 * R + r) * ESZ), me.z);
                S qw = zero_s<S>();
                for (int q = 0; q < L.P; ++q) {
                    const unsigned char *pr = tl + L.part() + L.part_bytes() * (q * R + r);
                    const int voff = reinterpret_cast<const int *>(pr)[0];
                    const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vals + voff + coff);
                    st[(2 * q) * 32 + lane] = live ? zwc_s(me.z, v.w) : zero_s<S>();
                    st[(2 * q + 1) * 32 + lane] = live ? zwc_s(v.z, me.w) : zero_s<S>();
                    if (want_tr) {
                        qz = add_s(qz, mul_s(lds_s<S>(pr + 16), v.z));
                        qw = add_s(qw, mul_s(lds_s<S>(pr + 16 + ESZ), conj_s(v.w)));
                    }
                }
                if (want_tr && live) tr = add_s(tr, add_s(zwc_s(qz, me.w), mul_s(me.z, qw)));
                __syncwarp();
                if (want_red) {
                    // one task per (record, row slot, group part): sum the chains, one RMW/RED
                    const int nt = (2 * L.P + 2) * R * gpr;
                    for (int tk = lane; tk < nt; tk += 32) {
                        const int q2 = tk / (R * gpr), rem = tk % (R * gpr);
                        const int r2 = rem / gpr, g2 = rem % gpr;
                        if (!(rs[R + r2] & 2)) continue;
                        int slot;
                        bool is_diag = false;
                        if (q2 < 2 * L.P) {
                            slot = reinterpret_cast<const int *>(tl + L.part() +
                                                                 L.part_bytes() * ((q2 >> 1) * R + r2))[1 + (q2 & 1)];
                        } else if (q2 == 2 * L.P) {
                            slot = rs[2 * R + r2];
                            is_diag = true;
                        } else {
                            slot = rs[3 * R + r2];
                        }
                        const int c0 = g2 * gse;
                        if (slot < 0 || cb + c0 >= p.chains) continue;
                        S sum = zero_s<S>();
                        for (int cc = 0; cc < gse; ++cc) sum = add_s(sum, st[q2 * 32 + r2 * C + c0 + cc]);
                        const int64_t grp = (cb + c0) / p.gs;
                        double *dst = is_diag ? p.slot_diag + (grp * p.n + slot) * (ESZ / 8)
                                              : p.slot_pat + (grp * p.pcount + slot) * (ESZ / 8);
                        if (p.gs > C) atomic_add_to(dst, sum);
                        else add_to(dst, sum);
                    }
                }
                __syncwarp();
            }
            if (lane == 0) mbar_arrive(smem_u32(&b_ddone[T % NGBUF]));
        }
        if (want_tr) {
            // trace: sum the lane registers over row slots and the chains of each group
            __syncwarp();
            st[lane] = active ? tr : zero_s<S>();
            __syncwarp();
            if (lane < gpr && cb + lane * gse < p.chains) {
                S sum = zero_s<S>();
                for (int r2 = 0; r2 < R; ++r2)
                    for (int cc = 0; cc < gse; ++cc) sum = add_s(sum, st[r2 * C + lane * gse + cc]);
                double *dst = p.slot_trace + (int64_t)((cb + lane * gse) / p.gs) * (ESZ / 8);
                if (p.gs > C) atomic_add_to(dst, sum);
                else add_to(dst, sum);
            }
        }
    } else {
        // ================= N: noise, steps T0 + w, T0 + w + NW, ...
        const int w = warp - 3;
        for (int64_t T = T0 + w; T < T_end; T += NW) {
            if (T - NQ >= T0) mbar_wait(smem_u32(&b_nempty[T % NQ]), par(T - NQ, T0, NQ));
            mbar_wait(smem_u32(&b_tile[T % NTILE]), par(T, T0, NTILE));
            const int *rs = reinterpret_cast<const int *>(tile_of(T) + 32);
            double phi = 0.0;
            if (rs[R + r] & 2) {
                if (p.noise == 0)
                    phi = gaussian(static_cast<uint32_t>(rs[r]), p.sweep_abs0 + static_cast<uint32_t>(T / S_n), gchain,
                                   p.key0, p.key1);
                else
                    phi = p.noise == 2 ? 1.0 : 0.0;
            }
            noise[(T % NQ) * 32 + lane] = phi;
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&b_nfull[T % NQ]));
        }
    }
}

template <typename S>
size_t sweep2_smem(int tile_slot, int max_parts) {
    constexpr int ESZ = sizeof(S);
    const size_t stage = (size_t)(2 * max_parts + 2) * 32 * ESZ;
    const size_t nbars = NTILE + 3 * NGBUF + 2 * NQ;
    return (size_t)ValueArea<ESZ>::BYTES + (size_t)NTILE * tile_slot + NQ * 32 * 8 + stage + nbars * 8;
}

template <typename S, int C, int R, int NW>
static cudaError_t launch2(const Sweep2Params<S> &p, cudaStream_t st) {
    const size_t smem = sweep2_smem<S>(p.tile_slot, p.max_items);
    cudaError_t e =
        cudaFuncSetAttribute(sweep2_kernel<S, C, R, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sweep2_kernel<S, C, R, NW><<<p.ld / C, 32 * (3 + NW), smem, st>>>(p);
    return cudaGetLastError();
}

template <typename S>
cudaError_t launch_sweep2(const Sweep2Params<S> &p, int C, cudaStream_t st) {
    switch (C) {
        case 8: return launch2<S, 8, 4, 2>(p, st);
        case 16: return launch2<S, 16, 2, 2>(p, st);
        default: return launch2<S, 32, 1, 2>(p, st);
    }
}

template cudaError_t launch_sweep2<double>(const Sweep2Params<double> &, int, cudaStream_t);
template cudaError_t launch_sweep2<cd>(const Sweep2Params<cd> &, int, cudaStream_t);
template size_t sweep2_smem<double>(int, int);
template size_t sweep2_smem<cd>(int, int);

}  // namespace mcinv
