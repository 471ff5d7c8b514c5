// sweep_common.cuh -- device helpers shared by the sweep kernels (sweep3.cu: v3
// level kernel and v4 dataflow kernel; sweep5.cu: v5 dataflow kernel with
// TMA-staged plan blocks): lane-group reductions, state addressing and 16/32-B
// state accesses, the Eq. (4)/(5) fma chains, posted slot reductions, the fused
// accumulation of Eq. (1/C) and the dataflow counter wait.
#pragma once
#include <cstdint>
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
    const int nlow = any ? static_cast<int>(static_cast<unsigned>(rec.z) >> 16) : 0;
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


// TMA bulk staging of plan blocks (v5, v6): mbarrier init / parity wait, and one
// cp.async.bulk global -> shared copy completing on an mbarrier.
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

}  // namespace

}  // namespace mcinv
