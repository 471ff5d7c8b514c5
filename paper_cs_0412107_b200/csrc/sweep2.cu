// sweep2.cu -- K1/K2 (v2): the CC sweep on a dependency-respecting step
// schedule (plan.h), warp-specialized.
//
// One CTA owns C chains; lanes = C chains x R row slots (C * R = 32). The
// planner guarantees that the rows of a step do not depend on each other and
// that every operand is exactly the one the sequential sweep (Eq. 4/5,
// PAPER.md:157-160) reads, so z and w are bit-identical to row-by-row order.
//
// Warp roles (all synchronised with mbarriers, per step slot):
//   A  (1 warp)   the serial part only: for each step, the fma chains of
//                 Eq. (4)/(5) over smem operands, z_i, w_i to HBM and to the
//                 16-step result ring, FULL-output snapshots.
//   B  (1 warp)   producer: TMA bulk copy of the record tile of step U+8
//                 (cols, coefficients, smem source offsets, accumulation
//                 records) and cp.async gathers of step U's far operands
//                 (>= 8 steps old) from the [n][ld] state in HBM.
//   D  (ND warps) accumulation (sampling sweeps): diag, pattern and trace
//                 products of the rows finished in the step (Eq. 1/C, Eq. tr,
//                 P:173-182), smem transpose-reduction over the chains of an
//                 SE group, one RMW (or RED) per group slot.
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

// phase parity of the u-th use of a step-indexed barrier slot (u = (T - T0) / nslots)
template <int NSLOTS>
__device__ __forceinline__ uint32_t par(uint32_t T, uint32_t T0) {
    return ((T - T0) / NSLOTS) & 1u;
}

}  // namespace

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
    unsigned char *stage0 = reinterpret_cast<unsigned char *>(noise + NQ * 32);  // ND x [2P+2][32] S
    const int stage_bytes = (2 * p.max_items + 2) * 32 * ESZ;
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage0 + (size_t)ND * stage_bytes);
    const uint32_t b_tile = smem_u32(bars);               // [NTILE] TMA complete_tx
    const uint32_t b_gather = b_tile + 8 * NTILE;         // [NGBUF] 32 cp.async arrivals
    const uint32_t b_adone = b_gather + 8 * NGBUF;        // [NGBUF] A finished step
    const uint32_t b_ddone = b_adone + 8 * NGBUF;         // [NGBUF] D finished step
    const uint32_t b_nfull = b_ddone + 8 * NGBUF;         // [NQ] noise ready
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
    const uint32_t tile_slot = (uint32_t)p.tile_slot;
    auto tile_of = [&](uint32_t T) { return tiles + (T % NTILE) * tile_slot; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NTILE; ++s) mbar_init(b_tile + 8 * s, 1);
        for (int s = 0; s < NGBUF; ++s) {
            mbar_init(b_gather + 8 * s, 32);
            mbar_init(b_adone + 8 * s, 1);
            mbar_init(b_ddone + 8 * s, 1);
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
        // ================= B: tiles and gathers
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
            if (U >= T0 + 8) mbar_wait(b_adone + 8 * (U % NGBUF), par<NGBUF>(U - 8, T0));
            if (U >= T0 + 7) mbar_wait(b_ddone + 8 * ((U - 7) % NGBUF), par<NGBUF>(U - 7, T0));
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
        // ================= A: the serial fma chains
        S acc_z = zero_s<S>(), acc_w = zero_s<S>();
        ZW<S> *zw_chain = p.zw + chain;
        const unsigned char *vlane = vals + coff;
        unsigned char *ring_lane = vals + roff + coff;
        for (uint32_t T = T0; T < T_end; ++T) {
            mbar_wait(b_gather + 8 * (T % NGBUF), par<NGBUF>(T, T0));
            const unsigned char *tl = tile_of(T);
            const int K = reinterpret_cast<const int *>(tl)[0];
            const TileLayout L{K, 0, R, ESZ};
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
            mbar_wait(b_nfull + 8 * (T % NQ), par<NQ>(T, T0));
            if (flags & 2) {
                const int row = reinterpret_cast<const int *>(tl + 32)[r];
                const double phi = noise[(T % NQ) * 32 + lane];
                const S dl = lds_s<S>(tl + L.dsq() + r * ESZ);
                const S sg = lds_s<S>(tl + L.dsq() + (R + r) * ESZ);
                const S zi = fma_s(neg_s(dl), acc_z, scale_s(sg, phi));
                const S wi = fma_s(neg_s(conj_s(dl)), acc_w, scale_s(conj_s(sg), phi));
                zw_chain[(int64_t)row * p.ld] = ZW<S>{zi, wi};
                *reinterpret_cast<ZW<S> *>(ring_lane + (T % NRING) * BLK) = ZW<S>{zi, wi};
                if (p.outputs & OUT_FULL) {
                    const uint32_t s_loc = T / S_n;
                    if ((int)s_loc >= p.burn_in) {
                        const int64_t t = (int64_t)s_loc - p.snap_s0;
                        p.snap_x[(t * p.n + row) * p.ld + chain] = zi;
                        p.snap_y[(t * p.n + row) * p.ld + chain] = wi;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(b_nempty + 8 * (T % NQ));
                mbar_arrive(b_adone + 8 * (T % NGBUF));
            }
        }
    } else if (warp > WB) {
        // ================= D: accumulation, steps T0 + dw, T0 + dw + ND, ...
        const int dw = warp - WB - 1;
        S *st = reinterpret_cast<S *>(stage0 + (size_t)dw * stage_bytes);
        const bool want_tr = (p.outputs & OUT_TRACE) != 0;
        const bool want_red = (p.outputs & (OUT_DIAG | OUT_PATTERN)) != 0;
        const int gse = p.gs < C ? p.gs : C;
        const int lg_gse = __ffs(gse) - 1;
        const int lg_tpr = 5 - lg_gse;          // tasks per record: 32 / gse
        const int lg_gpr = __ffs(C / gse) - 1;  // groups per row slot
        const bool use_atomic = p.gs > C || ND > 1;
        S tr = zero_s<S>();
        const unsigned char *vlane = vals + coff;
        for (uint32_t T = T0 + dw; T < T_end; T += ND) {
            mbar_wait(b_adone + 8 * (T % NGBUF), par<NGBUF>(T, T0));
            const uint32_t s_loc = T / S_n;
            if ((int)s_loc >= p.burn_in && (want_tr || want_red)) {
                const unsigned char *tl = tile_of(T);
                const int P = reinterpret_cast<const int *>(tl)[1];
                const TileLayout L{reinterpret_cast<const int *>(tl)[0], P, R, ESZ};
                const int *rs = reinterpret_cast<const int *>(tl + 32);
                const bool live = (rs[R + r] & 2) && active;
                const ZW<S> me = *reinterpret_cast<const ZW<S> *>(vlane + roff + (T % NRING) * BLK);
                const S self = live ? zwc_s(me.z, me.w) : zero_s<S>();
                st[(2 * P) * 32 + lane] = self;      // diag
                st[(2 * P + 1) * 32 + lane] = self;  // pattern (i,i)
                S qz = mul_s(lds_s<S>(tl + L.dsq() + (2 * R + r) * ESZ), me.z);
                S qw = zero_s<S>();
                const unsigned char *pr = tl + L.part() + L.part_bytes() * r;
                for (int q = 0; q < P; ++q, pr += L.part_bytes() * R) {
                    const ZW<S> v = *reinterpret_cast<const ZW<S> *>(vlane + reinterpret_cast<const int *>(pr)[0]);
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
                    // task = (record q2, row slot r2, group g2): sum gse chains, one RMW/RED
                    const int nt = (2 * P + 2) << lg_tpr;
                    for (int tk = lane; tk < nt; tk += 32) {
                        const int q2 = tk >> lg_tpr, rem = tk & ((1 << lg_tpr) - 1);
                        const int r2 = rem >> lg_gpr, g2 = rem & ((1 << lg_gpr) - 1);
                        if (!(rs[R + r2] & 2)) continue;
                        int slot;
                        double *base;
                        int64_t cnt;
                        if (q2 < 2 * P) {
                            slot = reinterpret_cast<const int *>(tl + L.part() +
                                                                 L.part_bytes() * ((q2 >> 1) * R + r2))[1 + (q2 & 1)];
                            base = p.slot_pat;
                            cnt = p.pcount;
                        } else if (q2 == 2 * P) {
                            slot = rs[2 * R + r2];
                            base = p.slot_diag;
                            cnt = p.n;
                        } else {
                            slot = rs[3 * R + r2];
                            base = p.slot_pat;
                            cnt = p.pcount;
                        }
                        const int c0 = g2 << lg_gse;
                        if (slot < 0 || cb + c0 >= p.chains) continue;
                        const S *sp = st + q2 * 32 + r2 * C + c0;
                        S sum = sp[0];
                        for (int cc = 1; cc < gse; ++cc) sum = add_s(sum, sp[cc]);
                        double *dst = base + (((int64_t)(cb + c0) / p.gs) * cnt + slot) * (ESZ / 8);
                        if (use_atomic) atomic_add_to(dst, sum);
                        else add_to(dst, sum);
                    }
                }
                __syncwarp();
            }
            if (lane == 0) mbar_arrive(b_ddone + 8 * (T % NGBUF));
        }
        if (want_tr) {
            // trace: sum the lane registers over row slots and the chains of each group
            __syncwarp();
            st[lane] = active ? tr : zero_s<S>();
            __syncwarp();
            const int gpr = C >> lg_gse;
            if (lane < gpr && cb + (lane << lg_gse) < p.chains) {
                S sum = zero_s<S>();
                for (int r2 = 0; r2 < R; ++r2)
                    for (int cc = 0; cc < gse; ++cc) sum = add_s(sum, st[r2 * C + (lane << lg_gse) + cc]);
                atomic_add_to(p.slot_trace + (int64_t)((cb + (lane << lg_gse)) / p.gs) * (ESZ / 8), sum);
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
    const size_t stage = (size_t)kND * (2 * max_parts + 2) * 32 * ESZ;
    const size_t nbars = NTILE + 3 * NGBUF + 2 * NQ;
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
