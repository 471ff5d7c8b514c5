// mcinv_host.cu -- the C ABI of include/mcinv.h: H1 host preprocessing,
// workspace layout, and the launch sequence of the hot path.
//
// Everything numeric on the hot path runs in the kernels of sweep.cu,
// contract.cu and reduce.cu. This file validates inputs, builds the device
// form of C (row/column union lists, 1/c_ii, 1/sqrt(c_ii)), lays out the
// workspace and enqueues kernels on the caller's stream.
#include <algorithm>
#include <complex>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <cstdlib>
#include <future>
#include <map>
#include <memory>
#include <tuple>
#include <type_traits>

#include "../../include/mcinv.h"
#include "mcinv_internal.cuh"
#include "levels.h"

using mcinv::cd;
using mcinv::ZW;

namespace {

// Device buffers come from the stream-ordered allocator (cudaMallocAsync on the
// legacy stream, default pool with an unlimited release threshold): creating and
// destroying contexts does not synchronize the device (cudaFree would), which
// matters for the end-to-end path (a context per matrix).
inline cudaError_t dev_alloc(void **p, size_t bytes) { return cudaMallocAsync(p, bytes, 0); }

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, 0);
        p = nullptr;
        bytes = 0;
    }
};

struct Entry {
    int j;
    std::complex<double> v;
};

// Device copy of the level schedule (levels.h) for the v3 kernel.
struct LevelDev {
    DevBuf ph_row, ord_rec, ent_col, ent_ab, ent_pz, ord_dsg;
    DevBuf ph_tq, tq_row, tq_eptr, tq_col, tq_val, ph_pp, pp_i, pp_j, pp_slot;
    int D = 0, max_rows = 0, ntq = 0;
    bool deferred = false;                   // deferred items exist (v4 / v6 cannot run this plan)
    bool deferred_pairs = false;             // deferred pattern pairs exist (v5 cannot run this plan)
    std::string error;
    mcinv::LevelPlan host;                   // kept only for mcinv_debug_levels
    std::vector<int4> h_rec;                 // level-order records, for the v4 slot arrays
    std::vector<unsigned char> h_dsg;        // level-order {delta, sigma} (raw bytes of S)
    std::vector<int> h_ph_row;
    std::vector<int> h_ent_col;              // level-order entry columns (v4 slot ordering)
    std::vector<unsigned char> h_ab;         // level-order {a, b} pairs (raw bytes of S), for v5 blocks
    std::vector<int> h_pz;                   // level-order pattern slot pairs (empty without pattern)
    std::vector<int> h_tq_row, h_tq_eptr, h_tq_col;  // trace items (v5 schedules them as dataflow items)
    std::vector<unsigned char> h_tq_val;     // their Q values (raw bytes of S)
    struct Slots {
        DevBuf rec, dsg;
        int nslots = 0;
        // v5: one contiguous block per warp group (records, delta/sigma, columns, coefficients,
        // pattern slots), staged into shared memory by a TMA bulk copy
        DevBuf blob, gofs;
        int maxb = 0;
        std::vector<int> h_x;           // host-only contexts (mcinv_debug_blocks): rec.x per slot
        std::vector<unsigned> h_mask;   // ... and its wait mask (v6 blocks)
    };
    // (rows per warp group R, warps W, TMA blocks, entry padding, block entry cap) -> slot arrays
    std::map<std::tuple<int, int, int, int, int>, std::unique_ptr<Slots>> slots;
};

struct Layout {
    int ver = 3;            // sweep kernel: 1 row-by-row, 2 step schedule, 3 level schedule
    int lgC = 0, lgP = 0;   // v3: log2 chains per CTA and per accumulator sub-slot
    int Gs = 0, ksub = 1;   // accumulator sub-slots (Gs = G * ksub)
    int ld = 0, G = 0, T = 0;
    int e = 1;              // doubles per scalar
    size_t zw = 0, slot_diag = 0, slot_pat = 0, slot_full = 0, slot_trace = 0, snap_x = 0, snap_y = 0, mom = 0;
    size_t series = 0;      // TRACE: Geyer's series [series_cap][e] (0 bytes when off)
    int64_t series_cap = 0;
    size_t mom_count = 0;   // doubles in the moment vector
    size_t mom_diag = 0, mom_pat = 0, mom_full = 0, mom_trace = 0;  // offsets (doubles) of S1 in moments
    size_t mom_m2 = 0;      // offset (doubles) of the M2 block: M2 of an output at mom_<output> + mom_m2
    size_t total = 0;
};

}  // namespace

struct mcinv_ctx {
    int device = 0;
    int dtype = MCINV_F64;
    int64_t n = 0;
    std::string err;
    int64_t err_index = -1;
    bool valid = false;
    bool host_only = false;  // mcinv_debug_levels: no device allocations

    // host canonical C (rows sorted, duplicates summed), kept for the default pattern
    std::vector<int64_t> h_rp;
    std::vector<int> h_col;
    // host copies for the level planner (levels.h)
    std::vector<int> h_u_ptr, h_u_col;
    std::vector<std::complex<double>> h_u_a, h_u_b, h_delta, h_sigma;
    std::vector<int> h_prow, h_pcol;
    std::vector<int64_t> h_q_ptr;
    std::vector<int> h_q_col;
    std::vector<std::complex<double>> h_q_val;
    std::map<unsigned, std::unique_ptr<LevelDev>> levels;                 // outputs -> level schedule
    int nsm = 148;
    int64_t l2_bytes = 126 << 20;  // device L2 (queried at create)
    mutable int depth = -1;        // levels D of the row DAG (cached by level_depth)
    int last_kernel = 0;  // 1 = v1 (row by row), 3 = v3 (level schedule), 4 = v4 (dataflow)
    DevBuf err_flag;      // v4 watchdog flag (device unsigned)
    int last_C = 0;
    int64_t last_steps = 0;
    int last_threads = 0, last_K = 1, last_blocks = 0;  // launch layout of the last sweep kernel
    // device C
    DevBuf u_ptr, u_col, u_a, u_b, delta, sigma;
    // pattern
    bool pattern_custom = false;
    int64_t pcount = 0;
    DevBuf p_ptr, p_idx, p_other;
    // Q
    bool have_q = false;
    DevBuf qr_ptr, qr_col, qr_val, qc_ptr, qc_row, qc_val;
    // last run
    bool have_run = false;
    int64_t acc_cycles = 0;  // sampling sweeps accumulated since the last fresh (non-resume) run
    mcinv_run_args last{};
    Layout lay;
    DevBuf own_ws;
    char *ws = nullptr;
    cudaStream_t stream = nullptr;
    DevBuf tmp;  // staging for host-side results
    DevBuf ozaki;  // K3 Ozaki scratch (int8 digit planes and exponents), MCINV_CONTRACT_OZAKI=1
    // instrumentation
    bool timing = false;
    int64_t launches = 0;
    struct Timed {
        cudaEvent_t a, b;
        int kind;  // 0 sweep, 1 contract
    };
    std::vector<Timed> pending;
    std::vector<cudaEvent_t> event_pool;
    ~mcinv_ctx() {
        for (auto &t : pending) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        for (auto e : event_pool) cudaEventDestroy(e);
    }
};

namespace {

mcinv_status fail(mcinv_ctx *c, mcinv_status st, const std::string &msg, int64_t idx = -1) {
    if (c) {
        c->err = msg;
        c->err_index = idx;
    }
    return st;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ctx, MCINV_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <typename T>
mcinv_status upload(mcinv_ctx *ctx, DevBuf &b, const std::vector<T> &h) {
    b.release();
    if (ctx->host_only) return MCINV_OK;
    const size_t bytes = std::max<size_t>(sizeof(T), h.size() * sizeof(T));
    if (dev_alloc(&b.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        return fail(ctx, MCINV_E_NOMEM, "device allocation failed");
    }
    b.bytes = bytes;
    // on the legacy stream, in order with the allocation; callers synchronize that
    // stream before the data is used on another stream (uploads_done)
    if (!h.empty()) CK(cudaMemcpyAsync(b.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, 0));
    return MCINV_OK;
}

#define TRY(x)                                  \
    do {                                        \
        mcinv_status s_ = (x);                  \
        if (s_ != MCINV_OK) return s_;          \
    } while (0)

// Validate a CSR and return canonical rows: sorted by column, duplicates summed.
mcinv_status read_csr(mcinv_ctx *ctx, int64_t n, const int64_t *rp, const int32_t *col, const double *val, bool cplx,
                      std::vector<std::vector<Entry>> &rows) {
    if (!rp || !col || !val) return fail(ctx, MCINV_E_INVALID, "null CSR pointer");
    if (rp[0] != 0) return fail(ctx, MCINV_E_INVALID, "row_ptr[0] != 0");
    for (int64_t i = 0; i < n; ++i)
        if (rp[i + 1] < rp[i]) return fail(ctx, MCINV_E_INVALID, "row_ptr decreasing", i);
    if (rp[n] >= (int64_t(1) << 31)) return fail(ctx, MCINV_E_INVALID, "nnz >= 2^31");
    rows.assign(n, {});
    for (int64_t i = 0; i < n; ++i) {
        auto &r = rows[i];
        r.reserve(rp[i + 1] - rp[i]);
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
            if (col[e] < 0 || col[e] >= n) return fail(ctx, MCINV_E_INVALID, "column out of range", i);
            const double re = cplx ? val[2 * e] : val[e], im = cplx ? val[2 * e + 1] : 0.0;
            if (!std::isfinite(re) || !std::isfinite(im)) return fail(ctx, MCINV_E_INVALID, "non-finite value", i);
            r.push_back(Entry{col[e], std::complex<double>(re, im)});
        }
        std::stable_sort(r.begin(), r.end(), [](const Entry &a, const Entry &b) { return a.j < b.j; });
        size_t o = 0;
        for (size_t q = 0; q < r.size(); ++q) {
            if (o > 0 && r[o - 1].j == r[q].j) r[o - 1].v += r[q].v;
            else r[o++] = r[q];
        }
        r.resize(o);
    }
    return MCINV_OK;
}

template <typename S> S to_s(std::complex<double> v);
template <> double to_s<double>(std::complex<double> v) { return v.real(); }
template <> cd to_s<cd>(std::complex<double> v) { return cd{v.real(), v.imag()}; }

// H1: C = L + D + U; union row/column lists; delta, sigma.
template <typename S>
mcinv_status build_matrix(mcinv_ctx *ctx, const std::vector<std::vector<Entry>> &rows) {
    const int64_t n = ctx->n;
    std::vector<std::complex<double>> diag(n);
    std::vector<std::vector<Entry>> colv(n);  // colv[i]: (j, c_ji) for j != i
    ctx->h_rp.assign(n + 1, 0);
    ctx->h_col.clear();
    for (int64_t i = 0; i < n; ++i) {
        bool have = false;
        for (const Entry &e : rows[i]) {
            ctx->h_col.push_back(e.j);
            if (e.j == i) {
                diag[i] = e.v;
                have = true;
            } else {
                colv[e.j].push_back(Entry{(int)i, e.v});  // rows ascend -> sorted
            }
        }
        ctx->h_rp[i + 1] = (int64_t)ctx->h_col.size();
        if (!have || diag[i] == std::complex<double>(0.0, 0.0))
            return fail(ctx, MCINV_E_ZERO_DIAG, "zero or missing diagonal", i);
        if (ctx->dtype == MCINV_F64 && !(diag[i].real() > 0.0))
            return fail(ctx, MCINV_E_DIAG_DOMAIN, "real path needs c_ii > 0", i);
    }
    std::vector<int> u_ptr(n + 1, 0), u_col;
    std::vector<S> u_a, u_b, dl(n), sg(n);
    u_col.reserve(2 * ctx->h_col.size());
    for (int64_t i = 0; i < n; ++i) {
        const auto &r = rows[i];
        const auto &c = colv[i];
        size_t p = 0, q = 0;
        while (p < r.size() || q < c.size()) {
            if (p < r.size() && r[p].j == i) {  // skip the diagonal
                ++p;
                continue;
            }
            const int jr = p < r.size() ? r[p].j : INT32_MAX;
            const int jc = q < c.size() ? c[q].j : INT32_MAX;
            const int j = std::min(jr, jc);
            std::complex<double> a(0.0, 0.0), b(0.0, 0.0);
            if (jr == j) a = r[p++].v;
            if (jc == j) b = std::conj(c[q++].v);
            u_col.push_back(j);
            u_a.push_back(to_s<S>(a));
            u_b.push_back(to_s<S>(b));
            ctx->h_u_a.push_back(a);
            ctx->h_u_b.push_back(b);
        }
        u_ptr[i + 1] = (int)u_col.size();
        // delta_i = 1/c_ii, sigma_i = 1/sqrt(c_ii), principal branch (reading R1)
        if (ctx->dtype == MCINV_F64) {
            const double d = diag[i].real();
            dl[i] = to_s<S>(std::complex<double>(1.0 / d, 0.0));
            sg[i] = to_s<S>(std::complex<double>(1.0 / std::sqrt(d), 0.0));
        } else {
            dl[i] = to_s<S>(1.0 / diag[i]);
            sg[i] = to_s<S>(1.0 / std::sqrt(diag[i]));
        }
    }
    ctx->h_u_ptr = u_ptr;
    ctx->h_u_col = u_col;
    ctx->h_delta.resize(n);
    ctx->h_sigma.resize(n);
    for (int64_t i = 0; i < n; ++i) {
        if (ctx->dtype == MCINV_F64) {
            ctx->h_delta[i] = 1.0 / diag[i].real();
            ctx->h_sigma[i] = 1.0 / std::sqrt(diag[i].real());
        } else {
            ctx->h_delta[i] = 1.0 / diag[i];
            ctx->h_sigma[i] = 1.0 / std::sqrt(diag[i]);
        }
    }
    TRY(upload(ctx, ctx->u_ptr, u_ptr));
    TRY(upload(ctx, ctx->u_col, u_col));
    TRY(upload(ctx, ctx->u_a, u_a));
    TRY(upload(ctx, ctx->u_b, u_b));
    TRY(upload(ctx, ctx->delta, dl));
    TRY(upload(ctx, ctx->sigma, sg));
    return MCINV_OK;
}

// Pattern lists keyed by r = max(i, j) (see DevPattern).
mcinv_status build_pattern(mcinv_ctx *ctx, int64_t count, const int32_t *rows, const int32_t *cols) {
    const int64_t n = ctx->n;
    std::vector<int> cnt(n + 1, 0), idx(std::max<int64_t>(count, 1)), other(std::max<int64_t>(count, 1));
    for (int64_t p = 0; p < count; ++p) {
        if (rows[p] < 0 || rows[p] >= n || cols[p] < 0 || cols[p] >= n)
            return fail(ctx, MCINV_E_INVALID, "pattern index out of range", p);
        cnt[std::max(rows[p], cols[p]) + 1]++;
    }
    for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<int> ptr(cnt.begin(), cnt.end()), fillp(cnt.begin(), cnt.end() - 1);
    for (int64_t p = 0; p < count; ++p) {
        const int r = rows[p], c = cols[p];
        const int at = fillp[std::max(r, c)]++;
        idx[at] = (int)p;
        // r >= c: z_r (current) conj(w_c); r < c: z_r (gathered) conj(w_c) at row c
        other[at] = (r >= c) ? c : (int)((unsigned)r | 0x80000000u);
    }
    idx.resize(std::max<int64_t>(count, 1));
    ctx->h_prow.assign(rows, rows + count);
    ctx->h_pcol.assign(cols, cols + count);
    ctx->levels.clear();
    TRY(upload(ctx, ctx->p_ptr, ptr));
    TRY(upload(ctx, ctx->p_idx, idx));
    TRY(upload(ctx, ctx->p_other, other));
    ctx->pcount = count;
    return MCINV_OK;
}

mcinv_status default_pattern(mcinv_ctx *ctx) {
    const int64_t n = ctx->n;
    std::vector<int32_t> r(ctx->h_col.size()), c(ctx->h_col.begin(), ctx->h_col.end());
    for (int64_t i = 0; i < n; ++i)
        for (int64_t e = ctx->h_rp[i]; e < ctx->h_rp[i + 1]; ++e) r[e] = (int32_t)i;
    return build_pattern(ctx, (int64_t)r.size(), r.data(), c.data());
}

template <typename S>
mcinv_status build_q(mcinv_ctx *ctx, const std::vector<std::vector<Entry>> &rows) {
    const int64_t n = ctx->n;
    std::vector<int> rptr(n + 1, 0), rcol, cptr(n + 1, 0), crow;
    std::vector<S> rval, cval;
    std::vector<std::vector<Entry>> colpart(n);
    ctx->h_q_ptr.assign(n + 1, 0);
    ctx->h_q_col.clear();
    ctx->h_q_val.clear();
    for (int64_t i = 0; i < n; ++i) {
        for (const Entry &e : rows[i]) {
            ctx->h_q_col.push_back(e.j);
            ctx->h_q_val.push_back(e.v);
        }
        ctx->h_q_ptr[i + 1] = (int64_t)ctx->h_q_col.size();
    }
    ctx->levels.clear();
    for (int64_t i = 0; i < n; ++i) {
        for (const Entry &e : rows[i]) {
            if (e.j <= i) {
                rcol.push_back(e.j);
                rval.push_back(to_s<S>(e.v));
            } else {
                colpart[e.j].push_back(Entry{(int)i, e.v});
            }
        }
        rptr[i + 1] = (int)rcol.size();
    }
    for (int64_t j = 0; j < n; ++j) {
        for (const Entry &e : colpart[j]) {
            crow.push_back(e.j);
            cval.push_back(to_s<S>(e.v));
        }
        cptr[j + 1] = (int)crow.size();
    }
    TRY(upload(ctx, ctx->qr_ptr, rptr));
    TRY(upload(ctx, ctx->qr_col, rcol));
    TRY(upload(ctx, ctx->qr_val, rval));
    TRY(upload(ctx, ctx->qc_ptr, cptr));
    TRY(upload(ctx, ctx->qc_row, crow));
    TRY(upload(ctx, ctx->qc_val, cval));
    ctx->have_q = true;
    return MCINV_OK;
}

cudaEvent_t get_event(mcinv_ctx *ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Launch a kernel-enqueueing callable, bracketing it with events when timing.
template <typename F>
void timed(mcinv_ctx *ctx, int kind, cudaStream_t st, F &&f) {
    ctx->launches++;
    if (!ctx->timing) {
        f();
        return;
    }
    mcinv_ctx::Timed t{get_event(ctx), get_event(ctx), kind};
    cudaEventRecord(t.a, st);
    f();
    cudaEventRecord(t.b, st);
    ctx->pending.push_back(t);
}

bool pow2_le32(int g) { return g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32; }

mcinv_status check_args(const mcinv_ctx *ctx_c, const mcinv_run_args *a) {
    mcinv_ctx *ctx = const_cast<mcinv_ctx *>(ctx_c);
    if (!a) return fail(ctx, MCINV_E_INVALID, "null args");
    if (a->chains < 1 || a->chain_begin < 0 || a->burn_in < 0 || a->cycles < 0 || a->sweep_begin < 0)
        return fail(ctx, MCINV_E_INVALID, "negative or empty run dimensions");
    if (!pow2_le32(a->group_size)) return fail(ctx, MCINV_E_INVALID, "group_size must be 1,2,4,8,16 or 32");
    if (a->chains % a->group_size || a->chain_begin % a->group_size)
        return fail(ctx, MCINV_E_INVALID, "chains and chain_begin must be multiples of group_size");
    if (a->chain_begin + a->chains > (int64_t(1) << 32) ||
        a->sweep_begin + a->burn_in + a->cycles > (int64_t(1) << 32))
        return fail(ctx, MCINV_E_INVALID, "chain or sweep index exceeds the 32-bit noise counter");
    if (a->outputs & ~15u) return fail(ctx, MCINV_E_INVALID, "unknown output bit");
    if ((a->outputs & MCINV_TRACE) && !ctx->have_q) return fail(ctx, MCINV_E_STATE, "TRACE needs mcinv_set_trace_q");
    if (a->noise < 0 || a->noise > 3) return fail(ctx, MCINV_E_INVALID, "noise mode");
    if (a->trace_series < 0 || a->trace_series > (int64_t(1) << 31))
        return fail(ctx, MCINV_E_INVALID, "trace_series capacity");
    if (a->chains > (int64_t(1) << 30)) return fail(ctx, MCINV_E_INVALID, "too many chains for one call");
    return MCINV_OK;
}

int kernel_pref() {  // 0 auto, 1 force v1, 3 force v3, 4 force v4, 5 force v5, 6 force v6
    const char *e = std::getenv("MCINV_KERNEL");
    if (!e) return 0;
    const char *d = e[0] == 'v' ? e + 1 : e;  // "v3" or "3"
    if (!std::strcmp(d, "1")) return 1;
    if (!std::strcmp(d, "3")) return 3;
    if (!std::strcmp(d, "4")) return 4;
    if (!std::strcmp(d, "5")) return 5;
    if (!std::strcmp(d, "6")) return 6;
    return 0;
}

int ilog2(int64_t x) {
    int l = 0;
    while ((int64_t(1) << (l + 1)) <= x) ++l;
    return l;
}

// v3: C = chains per CTA, the smallest power of two that fits the chains in
// one wave of CTAs (one per SM), at most 1024 (MCINV_C overrides)
// levels D of the lower-neighbour DAG (lev(i) = 1 + max lev of the lower neighbours), from the
// union adjacency; structure only, cached
int level_depth(const mcinv_ctx *ctx) {
    if (ctx->depth >= 0) return ctx->depth;
    std::vector<int> lev(ctx->n, 0);
    int D = 0;
    for (int64_t i = 0; i < ctx->n; ++i) {
        int l = 0;
        for (int q = ctx->h_u_ptr[i]; q < ctx->h_u_ptr[i + 1]; ++q)
            if (ctx->h_u_col[q] < i) l = std::max(l, lev[ctx->h_u_col[q]] + 1);
        lev[i] = l;
        D = std::max(D, l + 1);
    }
    ctx->depth = D;
    return D;
}

// chains per CTA: the smallest power of two that fits every chain in one wave of CTAs; for
// the level kernel (C > 32) rather the largest C from there down to 16 whose wave of CTAs
// keeps one level's state (rows per level x chains of the wave x sizeof(ZW)) in 3/4 of L2:
// the CTAs then run in several waves (each all sweeps of its chains) and the neighbours'
// lines of the previous levels hit L2 (config 5: C = 128 -> 16, 1.43 -> 1.62e10
// site-updates/s; config 4's levels are too wide for any C and keep C = 64)
int choose_lgC(const mcinv_ctx *ctx, int64_t chains) {
    if (const char *e = std::getenv("MCINV_C")) return ilog2(std::max(1, std::atoi(e)));
    int lg = 0;
    while (lg < 10 && ((chains + (int64_t(1) << lg) - 1) >> lg) > ctx->nsm) ++lg;
    if (lg <= 5 || std::getenv("MCINV_NO_L2_BLOCKING")) return lg;
    const double rows = (double)ctx->n / std::max(1, level_depth(ctx));
    const double zw = ctx->dtype == MCINV_C128 ? 32.0 : 16.0;
    for (int c = lg; c >= 4; --c) {
        const double wave_chains = std::min<double>((double)chains, (double)ctx->nsm * (double)(int64_t(1) << c));
        if (rows * wave_chains * zw <= 0.75 * (double)ctx->l2_bytes) return c;
    }
    return lg;
}

Layout make_layout(const mcinv_ctx *ctx, const mcinv_run_args *a) {
    Layout L;
    const int64_t n = ctx->n;
    const bool cplx = ctx->dtype == MCINV_C128;
    L.e = cplx ? 2 : 1;
    const size_t sz = 8 * L.e;
    L.ld = (int)((a->chains + 31) / 32 * 32);
    L.G = (int)(a->chains / a->group_size);
    const int pref = kernel_pref();
    L.ver = pref == 1 ? 1 : 3;  // v3 / v4 share the layout; run_typed picks v4 when eligible
    L.Gs = L.G;
    L.ksub = 1;
    if (L.ver == 3) {
        L.lgC = choose_lgC(ctx, a->chains);
        // (not capped at 32 for the dataflow kernels: config 4 measured 2.98e10 with v5 at
        // C = 32 vs 3.7e10 with v3 at C = 64 -- HBM-bound, the matrix row is read once per C)
        const int64_t q = std::max<int64_t>(32, int64_t(1) << L.lgC);  // padded chains stay in bounds
        L.ld = (int)((a->chains + q - 1) / q * q);
        // accumulator slots are the SE groups (the kernel sums the chains of a
        // group inside the CTA, then reduces into the group slot in L2)
        L.lgP = std::min(ilog2(a->group_size), L.lgC);  // lanes of one SE group inside a CTA
        L.ksub = 1;
        L.Gs = L.G;
    }
    L.T = 0;
    if (a->outputs & MCINV_FULL) {
        int T = a->snapshot_sweeps;
        if (T <= 0) {
            // K = T * gs >= 2048 per contraction (the A_g tiles are read and written once per
            // launch: the epilogue's share falls with K), at most 64 sweeps and 32 GB of
            // snapshots, bounded by cycles (T = 128 on config 3: contraction -3%, twice the memory)
            T = (int)std::max<int64_t>(1, 2048 / a->group_size);
            if (T > 64) T = 64;
            const int64_t per = 2 * n * (int64_t)L.ld * (int64_t)sz;
            while (T > 1 && T * per > (int64_t(32) << 30)) T /= 2;
        }
        if (a->cycles > 0 && T > a->cycles) T = (int)a->cycles;
        L.T = std::max(T, 1);
        // a resumed run keeps the snapshot chunk of the run it continues: the workspace
        // (and with it every offset) is then identical to the one the state lives in
        if (a->resume && ctx->have_run && ctx->lay.T > 0) L.T = ctx->lay.T;
    }
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align256(off + bytes);
        return o;
    };
    // state and accumulators first, the snapshot chunk (size T-dependent) last, so that
    // the offsets of everything a resumed run continues from do not depend on T
    L.zw = take((size_t)n * L.ld * 2 * sz);
    if (a->outputs & MCINV_DIAG) L.slot_diag = take((size_t)L.Gs * n * sz);
    if (a->outputs & MCINV_PATTERN) L.slot_pat = take((size_t)L.Gs * std::max<int64_t>(ctx->pcount, 1) * sz);
    if (a->outputs & MCINV_FULL) L.slot_full = take((size_t)L.G * n * n * sz);
    if (a->outputs & MCINV_TRACE) L.slot_trace = take((size_t)L.Gs * sz);
    if ((a->outputs & MCINV_TRACE) && a->trace_series > 0) {
        L.series_cap = a->trace_series;
        L.series = take((size_t)a->trace_series * sz);
    }
    size_t m = 0;
    // moment vector: S1 of every output, then M2 of every output (same order), then the
    // divergence count (mcinv_accumulators)
    if (a->outputs & MCINV_DIAG) { L.mom_diag = m; m += (size_t)n * L.e; }
    if (a->outputs & MCINV_PATTERN) { L.mom_pat = m; m += (size_t)ctx->pcount * L.e; }
    if (a->outputs & MCINV_FULL) { L.mom_full = m; m += (size_t)n * n * L.e; }
    if (a->outputs & MCINV_TRACE) { L.mom_trace = m; m += (size_t)L.e; }
    L.mom_m2 = m;
    L.mom_count = 2 * m + 1;
    L.mom = take(L.mom_count * 8);
    if (a->outputs & MCINV_FULL) {
        L.snap_x = take((size_t)L.T * n * L.ld * sz);
        L.snap_y = take((size_t)L.T * n * L.ld * sz);
    }
    L.total = off;
    return L;
}


// MCINV_HOST_TIMING=1: host planning phases to stderr (e2e diagnostics)
struct HostTimer {
    bool on = std::getenv("MCINV_HOST_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mcinv host] %-28s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

template <typename S>
LevelDev *get_levels(mcinv_ctx *ctx, unsigned outputs) {
    const unsigned key = outputs & (MCINV_PATTERN | MCINV_TRACE);
    auto it = ctx->levels.find(key);
    if (it != ctx->levels.end()) return it->second.get();
    std::unique_ptr<LevelDev> ld(new LevelDev());
    mcinv::LevelInput in;
    in.n = ctx->n;
    in.u_ptr = &ctx->h_u_ptr;
    in.u_col = &ctx->h_u_col;
    in.u_a = &ctx->h_u_a;
    in.u_b = &ctx->h_u_b;
    in.delta = &ctx->h_delta;
    in.sigma = &ctx->h_sigma;
    in.want_pattern = key & MCINV_PATTERN;
    in.want_trace = key & MCINV_TRACE;
    in.p_row = &ctx->h_prow;
    in.p_col = &ctx->h_pcol;
    in.q_ptr = &ctx->h_q_ptr;
    in.q_col = &ctx->h_q_col;
    in.q_val = &ctx->h_q_val;
    mcinv::LevelPlan &P = ld->host;
    HostTimer ht;
    ld->error = mcinv::build_levels(in, P);
    ht.mark("level plan");
    if (ld->error.empty()) {
        ld->D = P.D;
        ld->max_rows = P.max_rows;
        // entry arrays padded by 8 entries (col 0, zero coefficients, no pattern slot) so the
        // kernel's unrolled loads past a row's last entry stay in bounds
        const size_t ne = P.ent_col.size();
        P.ent_col.resize(ne + 8, 0);
        if (!P.ent_pz.empty()) P.ent_pz.resize(2 * (ne + 8), -1);
        std::vector<S> ab(2 * (ne + 8)), dsg(2 * ctx->n);
        for (size_t e = 0; e < ne; ++e) {
            ab[2 * e] = to_s<S>(P.ent_a[e]);
            ab[2 * e + 1] = to_s<S>(P.ent_b[e]);
        }
        for (int64_t o = 0; o < ctx->n; ++o) {
            dsg[2 * o] = to_s<S>(P.ord_dl[o]);
            dsg[2 * o + 1] = to_s<S>(P.ord_sg[o]);
        }
        // row record {i, entry begin, entries | lower entries << 16, pattern slot of (i,i)}
        std::vector<int4> rec(ctx->n);
        for (int64_t o = 0; o < ctx->n; ++o) {
            const int i = P.ord_row[o], beg = P.ord_eptr[o], cnt = P.ord_eptr[o + 1] - beg;
            int nlow = 0;
            while (nlow < cnt && P.ent_col[beg + nlow] < i) ++nlow;  // lower neighbours: a prefix
            if (cnt >= 65536) ld->error = "a row has 65536 or more off-diagonal entries";
            // packed in unsigned arithmetic (decoded as unsigned: nlow up to 65535)
            rec[o] = make_int4(i, beg, (int)((unsigned)cnt | (unsigned)nlow << 16), P.ord_pself[o]);
        }
        std::vector<S> tqv(P.tq_val.size());
        for (size_t e = 0; e < tqv.size(); ++e) tqv[e] = to_s<S>(P.tq_val[e]);
        mcinv_status st = MCINV_OK;
        auto up = [&](DevBuf &b, const auto &v) {
            if (st == MCINV_OK) st = upload(ctx, b, v);
        };
        up(ld->ph_row, P.ph_row);
        up(ld->ord_rec, rec);
        up(ld->ent_col, P.ent_col);
        up(ld->ent_ab, ab);
        up(ld->ord_dsg, dsg);
        up(ld->ent_pz, P.ent_pz);
        up(ld->ph_tq, P.ph_tq);
        up(ld->tq_row, P.tq_row);
        up(ld->tq_eptr, P.tq_eptr);
        up(ld->tq_col, P.tq_col);
        up(ld->tq_val, tqv);
        up(ld->ph_pp, P.ph_pp);
        up(ld->pp_i, P.pp_i);
        up(ld->pp_j, P.pp_j);
        up(ld->pp_slot, P.pp_slot);
        if (st != MCINV_OK && ld->error.empty()) ld->error = "level plan upload failed";
        ld->deferred = !P.pp_i.empty() || !P.tq_row.empty();
        ld->deferred_pairs = !P.pp_i.empty();
        ld->ntq = (int)P.tq_row.size();
        ld->h_rec = rec;
        ld->h_dsg.assign(reinterpret_cast<const unsigned char *>(dsg.data()),
                         reinterpret_cast<const unsigned char *>(dsg.data() + dsg.size()));
        ld->h_ph_row = P.ph_row;
        ld->h_ent_col = P.ent_col;
        ld->h_ab.assign(reinterpret_cast<const unsigned char *>(ab.data()),
                        reinterpret_cast<const unsigned char *>(ab.data() + ab.size()));
        ld->h_pz = P.ent_pz;
        ld->h_tq_row = P.tq_row;
        ld->h_tq_eptr = P.tq_eptr;
        ld->h_tq_col = P.tq_col;
        ld->h_tq_val.assign(reinterpret_cast<const unsigned char *>(tqv.data()),
                            reinterpret_cast<const unsigned char *>(tqv.data() + tqv.size()));
        if (!ctx->host_only) P = mcinv::LevelPlan();  // device copy only
    }
    LevelDev *raw = ld.get();
    ctx->levels[key] = std::move(ld);
    return raw;
}

// v4 slot arrays: level order with every level padded to a multiple of R rows
// (a warp group of R rows never spans two levels, so its rows are independent)
constexpr int kBlockEntries = 56;  // v5: entries per warp group (bounds the staged blocks)
int block_entries() {  // MCINV_BLOCK_ENTRIES overrides (experiments)
    const char *e = std::getenv("MCINV_BLOCK_ENTRIES");
    return e ? std::atoi(e) : kBlockEntries;
}
constexpr bool kV5Default = true;  // v5 by default where it applies (measured: config 2 +5%, config 3 +24%)
// v6 (two chains per thread) by default where it applies (MCINV_V6=0/1 overrides); its
// threads per CTA (MCINV_V6_THREADS)
bool v6_default() {  // config 2: 2.55 -> 2.77e10 site-updates/s over v5 (profiles/r02_v6*.log)
    const char *e = std::getenv("MCINV_V6");
    return e ? std::atoi(e) != 0 : true;
}
int v6_threads() {  // 512 (128 registers: the gathers of 4 entries of both chains in flight) measured best
    const char *e = std::getenv("MCINV_V6_THREADS");
    return e ? std::atoi(e) : 512;
}

// pad_ku: each row's entries in a block padded to a multiple of the kernel's gather unroll
// (0: the scalar type's default); ecap: entries per warp-group block (0: block_entries())
// wmask (v6): each row of a block also carries a 32-bit mask of the lower-neighbour
// entries it must wait for (see below)
template <typename S>
LevelDev::Slots *get_slots(mcinv_ctx *ctx, LevelDev *lv, int R, int W, bool blocks, int pad_ku = 0, int ecap = 0,
                           bool wmask = false) {
    if (ecap <= 0) ecap = block_entries();
    const int KU = pad_ku > 0 ? pad_ku : (sizeof(S) == sizeof(double) ? MCINV_V5_KUR : MCINV_V5_KUC);
    const auto key = std::make_tuple(R, W, (blocks ? 1 : 0) | (wmask ? 2 : 0), KU, ecap);
    auto it = lv->slots.find(key);
    if (it != lv->slots.end()) return it->second.get();
    std::unique_ptr<LevelDev::Slots> sl(new LevelDev::Slots());
    std::vector<int4> rec;
    std::vector<S> dsg;
    // v5 with trace: each trace item (Eq. tr, reading R2: conj(w_i) sum_j Q_ij z_j) joins the
    // schedule as a record that waits on rows i and j of its Q row (entries [i, Q cols..],
    // all waited for; coefficients {0, Q_ij}), is placed after them like a row after its
    // lower neighbours, and that no row waits on: record x = -2 - i
    const bool trace_items = blocks && !lv->h_tq_row.empty();
    std::vector<int4> xrec = lv->h_rec;
    std::vector<int> xcol = lv->h_ent_col;
    std::vector<unsigned char> xab = lv->h_ab;
    std::vector<int> xpz = lv->h_pz;
    std::vector<unsigned char> xdsg = lv->h_dsg;
    if (trace_items) {
        const S *qv = reinterpret_cast<const S *>(lv->h_tq_val.data());
        for (size_t t = 0; t < lv->h_tq_row.size(); ++t) {
            const int i = lv->h_tq_row[t], b = lv->h_tq_eptr[t], e = lv->h_tq_eptr[t + 1];
            const int cnt = 1 + (e - b);
            xrec.push_back(make_int4(-2 - i, (int)xcol.size(), (int)((unsigned)cnt | (unsigned)cnt << 16), -1));
            xcol.push_back(i);
            const ZW<S> zero{};
            xab.insert(xab.end(), reinterpret_cast<const unsigned char *>(&zero),
                       reinterpret_cast<const unsigned char *>(&zero) + sizeof(zero));
            for (int q = b; q < e; ++q) {
                xcol.push_back(lv->h_tq_col[q]);
                const ZW<S> c{qv[q], S{}};
                xab.insert(xab.end(), reinterpret_cast<const unsigned char *>(&c),
                           reinterpret_cast<const unsigned char *>(&c) + sizeof(c));
            }
            if (!xpz.empty()) xpz.insert(xpz.end(), 2 * (size_t)cnt, -1);
            xdsg.insert(xdsg.end(), 2 * sizeof(S), 0);
        }
    }
    const int64_t nrec = (int64_t)xrec.size();
    const S *hd = reinterpret_cast<const S *>(xdsg.data());
    HostTimer ht;
    // slot order: the list schedule (levels.h schedule_slots) with a slack of L = W groups
    // (the warps of a CTA); MCINV_SLOT_ORDER=level keeps plain level order (each level padded)
    const char *so = std::getenv("MCINV_SLOT_ORDER");
    // similarity window of the list schedule (levels.h): 64 measured best on config 2 (32: -2%,
    // 0: -4%; configs 3 and 5 unchanged; profiles/r02_schedule_knobs.log)
    const char *se = std::getenv("MCINV_SIMILAR");
    const int sim = se ? std::atoi(se) : 64;
    std::vector<int> order;
    if (so && !std::strcmp(so, "level")) {
        for (int l = 0; l < lv->D; ++l) {
            for (int o = lv->h_ph_row[l]; o < lv->h_ph_row[l + 1]; ++o) order.push_back(o);
            while (order.size() % R) order.push_back(-1);
        }
    } else if (const char *e = std::getenv("MCINV_SLACK")) {
        order = mcinv::schedule_slots(nrec, xrec, xcol, R, std::atoi(e), blocks ? ecap : 0, sim);
    } else {
        // the largest slack (W, 3W/4, W/2, 3W/8, ..., 1 groups) whose schedule pads at most
        // 5% of the slots (MCINV_SLACK_PAD, percent): wide DAGs (config 2: L = 24 of 32,
        // measured 2.26 -> 2.37e10 over the former 3% rule) take most of the slack, narrow
        // ones (lattices) less; if none does, the least padded one
        double pad = 5.0;
        if (const char *e = std::getenv("MCINV_SLACK_PAD")) pad = std::atof(e);
        std::vector<int> cand;
        for (int L = W; L >= 1; L /= 2) {
            cand.push_back(L);
            if (L >= 4 && (3 * L / 4) < L) cand.push_back(3 * L / 4);
        }
        // (the slack is chosen on schedules without the similarity window -- cheap, and the
        // candidates are scheduled concurrently on host threads -- and the final order is then
        // built once with it)
        std::vector<std::future<size_t>> sizes;
        for (int L : cand)
            sizes.push_back(std::async(std::launch::async, [&, L] {
                return mcinv::schedule_slots(nrec, xrec, xcol, R, L, blocks ? ecap : 0, 0).size();
            }));
        int chosen = 1;
        size_t best_size = 0;
        for (size_t k = 0; k < cand.size(); ++k) {
            const size_t sz = sizes[k].get();
            if ((double)sz <= (double)nrec * (1.0 + pad / 100.0)) {
                chosen = cand[k];
                for (size_t q = k + 1; q < cand.size(); ++q) sizes[q].wait();
                break;
            }
            if (best_size == 0 || sz < best_size) {
                best_size = sz;
                chosen = cand[k];
            }
        }
        ht.mark("slack candidates");
        order = mcinv::schedule_slots(nrec, xrec, xcol, R, chosen, blocks ? ecap : 0, sim);
    }
    ht.mark("list schedule");
    for (int o : order) {
        if (o < 0) {
            rec.push_back(make_int4(-1, 0, 0, -1));
            dsg.push_back(S{});
            dsg.push_back(S{});
        } else {
            rec.push_back(xrec[o]);
            dsg.push_back(hd[2 * o]);
            dsg.push_back(hd[2 * o + 1]);
        }
    }
    sl->nslots = (int)rec.size();
    if (upload(ctx, sl->rec, rec) != MCINV_OK || upload(ctx, sl->dsg, dsg) != MCINV_OK) return nullptr;
    if (blocks) {
        // group block: int4 head {EP, bytes, off_ab, off_pz}; int4 rec[R] {i, entry offset in
        // the block, count | lower << 16, pattern slot of (i,i)}; S dsg[R][2]; int col[EP];
        // ZW<S> ab[EP]; int2 pz[EP] (pattern runs). Each row's entries are padded to a multiple
        // of the kernel's gather unroll KU (4 real, 2 complex) with zero coefficients on the
        // row's last column (its own row if it has none): the unrolled fma chain then needs no
        // predicate, and fma(0, v, a) == a for the finite states of a converging run (only the
        // sign of an exact zero sum can differ). EP a multiple of 4; sections 16-B aligned.
        const bool pat = !xpz.empty();
        auto padded = [KU](int c) { return (c + KU - 1) / KU * KU; };
        const ZW<S> *hab = reinterpret_cast<const ZW<S> *>(xab.data());
        const size_t ng = rec.size() / R;
        // Wait masks (v6): row i must see its lower neighbours j final before its update.
        // Waiting on j is implied, and dropped, when (a) j is itself a lower neighbour of
        // another lower neighbour j' of i that i does wait on (j' published only after
        // seeing j final, or after its own implied waits: completion is transitive through
        // the release/acquire pairs of the counters), or (b) j sits in an earlier group of
        // the same warp in the slot schedule (program order of that warp). Bit e of the mask
        // covers lower entry e < 32; entries from 32 on are always waited for.
        std::vector<int> ord_of, grp_of;
        if (wmask) {
            ord_of.assign(ctx->n, -1);
            grp_of.assign(ctx->n, -1);
            for (int64_t o = 0; o < ctx->n; ++o) ord_of[lv->h_rec[o].x] = (int)o;
            for (size_t t = 0; t < order.size(); ++t)
                if (order[t] >= 0 && xrec[order[t]].x >= 0) grp_of[xrec[order[t]].x] = (int)(t / R);
        }
        auto lower_has = [&](int jp, int j) {  // is j a lower neighbour of jp?
            const int4 r = lv->h_rec[ord_of[jp]];
            const int nl = (int)((unsigned)r.z >> 16);
            const int *b = lv->h_ent_col.data() + r.y;
            return std::binary_search(b, b + nl, j);
        };
        const char *wm_env = std::getenv("MCINV_WAITMASK");  // 0: wait on every lower neighbour (A/B)
        const bool prune = !(wm_env && std::atoi(wm_env) == 0);
        auto wait_mask = [&](const int4 q) -> unsigned {
            const int nl = (int)((unsigned)q.z >> 16);
            if (!prune) return nl >= 32 ? 0xffffffffu : (1u << nl) - 1u;
            const int *cols = lv->h_ent_col.data() + q.y;
            std::vector<int> kept;
            unsigned m = 0;
            for (int e = nl - 1; e >= 0; --e) {
                const int j = cols[e];
                bool implied = e < 32 && grp_of[j] < grp_of[q.x] && (grp_of[j] % W) == (grp_of[q.x] % W);
                for (size_t k = 0; !implied && e < 32 && k < kept.size(); ++k) implied = lower_has(kept[k], j);
                if (!implied) {
                    kept.push_back(j);
                    if (e < 32) m |= 1u << e;
                }
            }
            return m;
        };
        const size_t mask_bytes = wmask ? ((size_t)4 * R + 15) / 16 * 16 : 0;
        std::vector<int64_t> gofs(ng + 1, 0);
        std::vector<unsigned char> blob;
        for (size_t g = 0; g < ng; ++g) {
            int E = 0;
            for (int r = 0; r < R; ++r)
                if (rec[g * R + r].x != -1) E += padded(rec[g * R + r].z & 0xffff);
            const int EP = (E + 3) / 4 * 4;
            const size_t off_wm = 16 + 16 * (size_t)R + 2 * sizeof(S) * R;  // masks (wmask) before the columns
            const size_t off_col = off_wm + mask_bytes;
            const size_t off_ab = off_col + 4 * (size_t)EP;
            const size_t off_pz = off_ab + sizeof(ZW<S>) * EP;
            const size_t bytes = (off_pz + (pat ? 8 * (size_t)EP : 0) + 15) / 16 * 16;
            const size_t base = blob.size();
            blob.resize(base + bytes, 0);
            unsigned char *b = blob.data() + base;
            reinterpret_cast<int4 *>(b)[0] = make_int4(EP, (int)bytes, (int)off_ab, (int)off_pz);
            int e = 0;
            for (int r = 0; r < R; ++r) {
                const int4 q = rec[g * R + r];
                const int cnt = q.x != -1 ? q.z & 0xffff : 0;  // rows and trace items carry entries
                reinterpret_cast<int4 *>(b + 16)[r] = make_int4(q.x, e, q.x != -1 ? q.z : 0, q.w);
                reinterpret_cast<S *>(b + 16 + 16 * R)[2 * r] = dsg[2 * (g * R + r)];
                reinterpret_cast<S *>(b + 16 + 16 * R)[2 * r + 1] = dsg[2 * (g * R + r) + 1];
                const unsigned wm_r = (wmask && q.x >= 0) ? wait_mask(q) : 0u;
                if (wmask) reinterpret_cast<unsigned *>(b + off_wm)[r] = wm_r;
                if (ctx->host_only) {
                    sl->h_x.push_back(q.x);
                    sl->h_mask.push_back(wm_r);
                }
                for (int t = 0; t < cnt; ++t) {
                    reinterpret_cast<int *>(b + off_col)[e + t] = xcol[q.y + t];
                    reinterpret_cast<ZW<S> *>(b + off_ab)[e + t] = hab[q.y + t];
                    if (pat) {
                        reinterpret_cast<int2 *>(b + off_pz)[e + t] = make_int2(xpz[2 * (q.y + t)], xpz[2 * (q.y + t) + 1]);
                    }
                }
                const int last = cnt > 0 ? xcol[q.y + cnt - 1] : (q.x >= 0 ? q.x : 0);
                for (int t = cnt; t < padded(cnt); ++t) {
                    reinterpret_cast<int *>(b + off_col)[e + t] = last;  // ab[e + t] stays zero
                    if (pat) reinterpret_cast<int2 *>(b + off_pz)[e + t] = make_int2(-1, -1);
                }
                e += padded(cnt);
            }
            for (int t = e; t < EP; ++t)
                if (pat) reinterpret_cast<int2 *>(b + off_pz)[t] = make_int2(-1, -1);
            sl->maxb = std::max(sl->maxb, (int)bytes);
            gofs[g + 1] = (int64_t)blob.size();
        }
        ht.mark("blocks + wait masks");
        if (upload(ctx, sl->blob, blob) != MCINV_OK || upload(ctx, sl->gofs, gofs) != MCINV_OK) return nullptr;
        ht.mark("upload");
    }
    LevelDev::Slots *raw = sl.get();
    lv->slots[key] = std::move(sl);
    return raw;
}

// K4 for every output of a run: S1 and M2 (about the local groups' mean, or with center
// about the global mean center[S1 offset] / center_G: mcinv_recenter)
void launch_all_moments(mcinv_ctx *ctx, const Layout &L, char *ws, unsigned outputs, const double *center,
                        double center_G, cudaStream_t st) {
    const int64_t n = ctx->n;
    const int e = L.e;
    double *mom = (double *)(ws + L.mom);
    auto one = [&](const void *slot, int k, int64_t comps, size_t off) {
        mcinv::launch_moments((const double *)slot, L.G, k, comps, mom + off, mom + off + L.mom_m2,
                              center ? center + off : nullptr, center_G, st);
        ctx->launches++;
    };
    if (outputs & MCINV_DIAG) one(ws + L.slot_diag, L.ksub, n * e, L.mom_diag);
    if (outputs & MCINV_PATTERN) one(ws + L.slot_pat, L.ksub, ctx->pcount * e, L.mom_pat);
    if (outputs & MCINV_FULL) one(ws + L.slot_full, 1, n * n * e, L.mom_full);
    if (outputs & MCINV_TRACE) one(ws + L.slot_trace, L.ksub, e, L.mom_trace);
}

template <typename S>
mcinv_status run_typed(mcinv_ctx *ctx, const mcinv_run_args *a, const Layout &L, char *ws, cudaStream_t st) {
    using namespace mcinv;
    const int64_t n = ctx->n;
    SweepParams<S> p{};
    p.A = DevMatrix<S>{(int)n, (const int *)ctx->u_ptr.p, (const int *)ctx->u_col.p, (const S *)ctx->u_a.p,
                       (const S *)ctx->u_b.p, (const S *)ctx->delta.p, (const S *)ctx->sigma.p};
    p.P = DevPattern{(int)ctx->pcount, (const int *)ctx->p_ptr.p, (const int *)ctx->p_idx.p,
                     (const int *)ctx->p_other.p};
    if (ctx->have_q)
        p.Q = DevQ<S>{(const int *)ctx->qr_ptr.p, (const int *)ctx->qr_col.p, (const S *)ctx->qr_val.p,
                      (const int *)ctx->qc_ptr.p, (const int *)ctx->qc_row.p, (const S *)ctx->qc_val.p};
    p.zw = reinterpret_cast<ZW<S> *>(ws + L.zw);
    p.ld = L.ld;
    p.chains = (int)a->chains;
    p.chain0 = (uint32_t)a->chain_begin;
    p.key0 = (uint32_t)a->seed;
    p.key1 = (uint32_t)(a->seed >> 32);
    p.noise = a->noise;
    p.sweep_abs0 = (uint32_t)a->sweep_begin;
    p.burn_in = (int)a->burn_in;
    p.outputs = a->outputs & ~(unsigned)MCINV_FULL;
    p.gs = a->group_size;
    p.G = L.G;
    p.slot_diag = (double *)(ws + L.slot_diag);
    p.slot_pat = (double *)(ws + L.slot_pat);
    p.slot_trace = (double *)(ws + L.slot_trace);
    const int total = (int)(a->burn_in + a->cycles);
    // divergence count: the last double of the moment vector, incremented by the sweep kernels
    // (every stored value is checked: reading R12's per-sweep rule); kept across resumes
    double *const mom = (double *)(ws + L.mom);
    p.bad = mom + L.mom_count - 1;

    if (!a->resume) {
        CK(cudaMemsetAsync(p.bad, 0, sizeof(double), st));
        CK(cudaMemsetAsync(ws + L.zw, 0, (size_t)n * L.ld * sizeof(ZW<S>), st));
        if (a->outputs & MCINV_DIAG) CK(cudaMemsetAsync(p.slot_diag, 0, (size_t)L.Gs * n * sizeof(S), st));
        if (a->outputs & MCINV_PATTERN)
            CK(cudaMemsetAsync(p.slot_pat, 0, (size_t)L.Gs * std::max<int64_t>(ctx->pcount, 1) * sizeof(S), st));
        if (a->outputs & MCINV_FULL) CK(cudaMemsetAsync(ws + L.slot_full, 0, (size_t)L.G * n * n * sizeof(S), st));
        if (a->outputs & MCINV_TRACE) CK(cudaMemsetAsync(p.slot_trace, 0, (size_t)L.Gs * sizeof(S), st));
        if (L.series_cap) CK(cudaMemsetAsync(ws + L.series, 0, (size_t)L.series_cap * sizeof(S), st));
    }
    // Geyer's series: sampling sweeps since the fresh run index it; it must hold them all
    const int64_t series_base = a->resume ? ctx->acc_cycles : 0;
    if (L.series_cap && series_base + a->cycles > L.series_cap)
        return fail(ctx, MCINV_E_INVALID, "trace_series capacity below the sampling sweeps", L.series_cap);
    p.series = L.series_cap ? (double *)(ws + L.series) : nullptr;
    p.series_base = (int)series_base;
    // kernel choice (Layout::ver): v3 level schedule (default), v1 row by row
    LevelDev *lv = L.ver == 3 ? get_levels<S>(ctx, a->outputs) : nullptr;
    if (lv && !lv->error.empty()) return fail(ctx, MCINV_E_INVALID, "level schedule: " + lv->error);
    if (lv && L.lgP > L.lgC) return fail(ctx, MCINV_E_INVALID, "layout: group lanes exceed chains per CTA");
    // dataflow kernels (v5 TMA-staged plan blocks, v4 plan through L1) when the chains of a
    // row fit one warp and the plan has no deferred items (trace, non-neighbour pairs); v5
    // when its shared memory (counters: a byte per row, a bit beyond 160k rows; two block
    // slots per warp) fits, else v4 when its byte counters fit (n <= 200k), else v3.
    // MCINV_KERNEL=v3|v4|v5 forces one (error if it does not apply).
    const int pref = kernel_pref();
    // v5 also runs trace items (as a phase after each sampling sweep); v4 / v6 need a plan
    // without deferred items
    const bool trace_flow = lv && L.lgC <= 5 && lv->deferred && !lv->deferred_pairs;
    const bool flow_ok = lv && L.lgC <= 5 && (!lv->deferred || (trace_flow && pref != 4 && pref != 6));
    if ((pref == 4 || pref == 5 || pref == 6) && !flow_ok)
        return fail(ctx, MCINV_E_INVALID, "dataflow kernel not applicable to this run");
    // v6 (v5 with the two chains of a Box-Muller pair per thread): real C, at least 2 chains
    // per CTA, both chains of a thread in one SE group (group_size >= 2: even chain_begin)
    const bool v6_ok = flow_ok && !lv->deferred && ctx->dtype == MCINV_F64 && L.lgC >= 1 && L.lgP >= 1 &&
                       a->group_size >= 2;
    if (pref == 6 && !v6_ok) return fail(ctx, MCINV_E_INVALID, "v6 kernel not applicable to this run");
    // auto: dataflow only up to 200k rows -- beyond, v3 (level barriers, K = 2 chains per
    // thread) measured 15-20% faster than v5 with bit counters at n = 1e6 (C = 8/16/32:
    // 3.04/3.45/3.69e10 vs 2.64/2.57/3.00e10 site-updates/s; profiles/r01_bigsmall.log)
    bool v4 = flow_ok && (pref == 4 || pref == 5 || pref == 6 || (pref == 0 && n <= 200000));  // v4, v5 or v6
    // chains per thread K (register blocking; real C, both chains in one SE group, no
    // trace / deferred items): default 2 for v3 (config 4 +19%), 1 for the dataflow kernels
    // (config 2 measured faster with more threads than with blocking, profiles/); MCINV_K
    int lgK = (lv && ctx->dtype == MCINV_F64 && L.lgC >= 1 && a->group_size >= 2 && !lv->deferred) ? 1 : 0;
    if (const char *e = std::getenv("MCINV_K")) lgK = std::atoi(e) >= 2 ? lgK : 0;
    if (v4) lgK = 0;
    // threads: v3 enough for the widest phase x C/K, at most 1024 (64 registers; measured
    // over 768 / 85 registers after the round's tuning: config 4 3.97 -> 4.15e10, config 5
    // 1.38 -> 1.43e10); dataflow 1024 real / 768 complex (more warps keep more rows in
    // flight; measured best for configs 2 / 3), fewer for tiny n; a multiple of 32 and of C/K
    auto threads_for = [&](bool flow) {
        int64_t want = flow ? std::min<int64_t>(ctx->dtype == MCINV_C128 ? 768 : 1024, (int64_t)n << (L.lgC - lgK))
                            : std::min<int64_t>(1024, (int64_t)std::max(lv->max_rows, 1) << (L.lgC - lgK));
        if (const char *e = std::getenv("MCINV_THREADS")) want = std::atoi(e);
        want = std::min<int64_t>(1024, std::max<int64_t>(want, int64_t(1) << (L.lgC - lgK)));
        return (int)((want + 31) / 32 * 32);
    };
    int threads3 = lv ? threads_for(v4) : 0;
    bool v6 = v4 && v6_ok && (pref == 6 || (pref == 0 && v6_default()));
    LevelDev::Slots *sl = nullptr;
    if (v6) {
        // R = 64 / C rows per warp group (C / 2 lanes per row); each row's entries padded to
        // the kernel's gather unroll; the block entry cap scaled with R, within the
        // shared-memory budget of two block slots per warp next to the counters
        if (!std::getenv("MCINV_THREADS")) threads3 = v6_threads();
        const int R = 64 >> L.lgC, W = threads3 / 32, ku = mcinv::sweep6_ku(threads3);
        const size_t counters = n > mcinv::kByteCounters ? ((size_t)n + 127) / 128 * 16 : ((size_t)n + 15) / 16 * 16;
        // shared-memory budget of one CTA (MCINV_V6_SMEM_KB: smaller budgets let several CTAs share an SM)
        long smem_budget = 220 * 1024;
        if (const char *e = std::getenv("MCINV_V6_SMEM_KB")) smem_budget = std::atol(e) * 1024;
        const long budget = (smem_budget - (long)counters) / (2 * W) - 16 - 36 * R - 64;
        int ecap = std::max(8, std::min<int>(block_entries() * R / 4, (int)(budget / 28)));
        if (const char *e = std::getenv("MCINV_BLOCK_ENTRIES")) ecap = std::atoi(e);
        // the cap counts unpadded entries: shrink it until the padded blocks fit
        for (int tries = 0; tries < 6; ++tries, ecap = std::max(8, ecap * 3 / 4)) {
            sl = get_slots<S>(ctx, lv, R, W, true, ku, ecap, true);
            if (!sl || mcinv::sweep6_smem((int)n, threads3, sl->maxb) <= 227 * 1024) break;
        }
        if (sl && mcinv::sweep6_smem((int)n, threads3, sl->maxb) > 227 * 1024) {
            if (pref == 6) return fail(ctx, MCINV_E_INVALID, "v6 blocks do not fit shared memory");
            v6 = false;
            sl = nullptr;
            threads3 = threads_for(v4);
        }
    }
    bool v5 = v4 && !v6 && (pref == 5 || (pref == 0 && kV5Default));
    if (v5) sl = get_slots<S>(ctx, lv, 32 >> L.lgC, threads3 / 32, true);
    if (v5 && sl && mcinv::sweep5_smem((int)n, threads3, sl->maxb) > 227 * 1024) {
        if (pref == 5) return fail(ctx, MCINV_E_INVALID, "v5 blocks do not fit shared memory");
        v5 = false;
    }
    if (v6) lgK = 1;
    if (v4 && !v5 && !v6 && lv->deferred) {  // trace items need v5 (its smem did not fit): level kernel
        if (pref == 5) return fail(ctx, MCINV_E_INVALID, "v5 blocks do not fit shared memory");
        v4 = false;
        threads3 = threads_for(false);
    }
    if (v4 && !v5 && !v6) {
        if (n > 200000) {  // v4's byte counters do not fit: level kernel (its layout is the same)
            if (pref == 4) return fail(ctx, MCINV_E_INVALID, "v4 counters do not fit shared memory");
            v4 = false;
            if (ctx->dtype == MCINV_F64 && L.lgC >= 1 && a->group_size >= 2 && !std::getenv("MCINV_K")) lgK = 1;
            threads3 = threads_for(false);
        } else {
            sl = get_slots<S>(ctx, lv, 32 >> L.lgC, threads3 / 32, false);
        }
    }
    if (!ctx->host_only) CK(cudaStreamSynchronize(0));  // plan uploads (legacy stream) complete
    if (v4 && !sl) return fail(ctx, MCINV_E_NOMEM, "v4 slot arrays");
    if (v4 && !ctx->err_flag.p) {
        if (dev_alloc(&ctx->err_flag.p, 16) != cudaSuccess) return fail(ctx, MCINV_E_NOMEM, "v4 flag");
        CK(cudaStreamSynchronize(0));
        ctx->err_flag.bytes = 16;
    }
    if (v4) CK(cudaMemsetAsync(ctx->err_flag.p, 0, 16, st));
    ctx->last_kernel = v6 ? 6 : v5 ? 5 : v4 ? 4 : L.ver;
    ctx->last_C = lv ? (1 << L.lgC) : 32;
    ctx->last_steps = lv ? lv->D : n;
    ctx->last_K = 1 << lgK;
    ctx->last_threads = lv ? threads3 : 0;
    ctx->last_blocks = lv ? (int)((a->chains + (int64_t(1) << L.lgC) - 1) >> L.lgC) : 0;
    Sweep3Params<S> q3{};
    if (lv) {
        q3.ph_row = (const int *)lv->ph_row.p;
        q3.ord_rec = (const int4 *)lv->ord_rec.p;
        q3.ent_col = (const int *)lv->ent_col.p;
        q3.ent_ab = (const S *)lv->ent_ab.p;
        q3.ent_pz = (const int2 *)lv->ent_pz.p;
        q3.ord_dsg = (const S *)lv->ord_dsg.p;
        q3.ph_tq = (const int *)lv->ph_tq.p;
        q3.tq_row = (const int *)lv->tq_row.p;
        q3.tq_eptr = (const int *)lv->tq_eptr.p;
        q3.tq_col = (const int *)lv->tq_col.p;
        q3.tq_val = (const S *)lv->tq_val.p;
        q3.ph_pp = (const int *)lv->ph_pp.p;
        q3.pp_i = (const int *)lv->pp_i.p;
        q3.pp_j = (const int *)lv->pp_j.p;
        q3.pp_slot = (const int *)lv->pp_slot.p;
        q3.D = lv->D;
        q3.zw = p.zw;
        q3.n = (int)n;
        q3.ld = L.ld;
        q3.chains = p.chains;
        q3.chain0 = p.chain0;
        q3.key0 = p.key0;
        q3.key1 = p.key1;
        q3.noise = p.noise;
        q3.sweep_abs0 = p.sweep_abs0;
        q3.burn_in = p.burn_in;
        q3.lgC = L.lgC;
        q3.lgG = ilog2(a->group_size);
        q3.lgK = lgK;
        q3.lgP = L.lgP - lgK;
        q3.pcount = (int)ctx->pcount;
        q3.slot_diag = p.slot_diag;
        q3.slot_pat = p.slot_pat;
        q3.slot_trace = p.slot_trace;
        q3.bad = p.bad;
        q3.series = p.series;
        q3.series_base = p.series_base;
        // MCINV_RECONV bits: 1 reconverge the warp at the end of each item (default: diag-only
        // config 2 1.57 -> 2.79e10), 2 also after the dependency waits (measured -6%)
        q3.reconv = 1;
        if (const char *e = std::getenv("MCINV_RECONV")) q3.reconv = std::atoi(e);
        if (sl) {
            q3.slot_rec = (const int4 *)sl->rec.p;
            q3.slot_dsg = (const S *)sl->dsg.p;
            q3.nslots = sl->nslots;
            q3.err = (unsigned *)ctx->err_flag.p;
            q3.blob = (const unsigned char *)sl->blob.p;
            q3.gofs = (const int64_t *)sl->gofs.p;
            q3.maxb = sl->maxb;
            // MCINV_SPIN_NS: nanosleep between counter polls; busy polling measured +1% config 2,
            // +3.6% config 3 over 32 ns (profiles/r01_spin.log)
            q3.spin_ns = 0;
            if (const char *e = std::getenv("MCINV_SPIN_NS")) q3.spin_ns = std::atoi(e);
            // MCINV_PREFETCH: L2 prefetch of every neighbour's line before the noise (3, default;
            // 220-sweep runs: config 2 2.02 -> 2.06e10, config 3 3.00 -> 3.26e10), upper
            // neighbours only into L2 (2) or L1 (1), none (0) -- profiles/r01_prefetch.log
            q3.prefetch = 3;
            // v6: the later gather chunks' lines with an L1 prefetch (+8: +1% on config 2,
            // profiles/r02_v6_stage.log)
            if (v6) q3.prefetch |= 8;
        }
        // v3 (level kernel): the same prefetch for real C (config 4: 3.82 -> 4.02e10), not for
        // complex (config 5: 1.36 -> 1.34e10)
        if (!sl && ctx->dtype == MCINV_F64) q3.prefetch = 3;
        if (const char *e = std::getenv("MCINV_PREFETCH")) q3.prefetch = std::atoi(e);
    }
    cudaError_t lerr = cudaSuccess;
    auto sweep = [&](int s0, int s1, int snap_s0, unsigned outs) {
        if (lv) {
            Sweep3Params<S> q = q3;
            q.s_begin = s0;
            q.s_end = s1;
            q.snap_s0 = snap_s0;
            q.outputs = outs;
            q.snap_x = (S *)(ws + L.snap_x);
            q.snap_y = (S *)(ws + L.snap_y);
            timed(ctx, 0, st, [&] {
                cudaError_t e;
                if constexpr (std::is_same<S, double>::value) {
                    if (v6) e = launch_sweep6(q, threads3, st);
                    else e = v5 ? launch_sweep5<S>(q, threads3, st)
                            : v4 ? launch_sweep4<S>(q, threads3, st) : launch_sweep3<S>(q, threads3, st);
                } else {
                    e = v5 ? launch_sweep5<S>(q, threads3, st)
                           : v4 ? launch_sweep4<S>(q, threads3, st) : launch_sweep3<S>(q, threads3, st);
                }
                if (e != cudaSuccess) lerr = e;
            });
        } else {
            SweepParams<S> q = p;
            q.s_begin = s0;
            q.s_end = s1;
            q.snap_s0 = snap_s0;
            q.outputs = outs;
            q.snap_x = (S *)(ws + L.snap_x);
            q.snap_y = (S *)(ws + L.snap_y);
            timed(ctx, 0, st, [&] { launch_sweep<S>(q, st); });
        }
    };
    if (!(a->outputs & MCINV_FULL)) {
        if (total > 0) sweep(0, total, 0, a->outputs);
    } else {
        // burn-in in one launch, then T-sweep chunks each followed by the
        // X Y^dagger contraction of its snapshots (MCINV_CONTRACT_OZAKI=1: the Ozaki scheme on
        // the tcgen05 int8 tensor cores, contract_ozaki.cu)
        // default for n >= 256 (config 3: the contraction 402 -> 320 ms per 64 sampling sweeps over
        // the TMA-fed DMMA kernel, profiles/r02_k3_ozaki.log); small n keeps DMMA (fewer launches)
        bool ozaki = n >= 256;
        if (const char *oz = std::getenv("MCINV_CONTRACT_OZAKI")) ozaki = std::atoi(oz) != 0;
        if (ozaki) {
            const size_t need = mcinv::contract_ozaki_scratch((int)n, L.T * a->group_size, ctx->dtype == MCINV_C128,
                                                                (int)(a->chains / a->group_size));
            if (ctx->ozaki.bytes < need) {
                ctx->ozaki.release();
                if (dev_alloc(&ctx->ozaki.p, need) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
                    cudaGetLastError();
                    ctx->ozaki.p = nullptr;
                    ozaki = false;
                } else {
                    ctx->ozaki.bytes = need;
                }
            }
        }
        if (a->burn_in > 0) sweep(0, (int)a->burn_in, 0, a->outputs & ~(unsigned)MCINV_FULL);
        for (int s0 = (int)a->burn_in; s0 < total; s0 += L.T) {
            const int s1 = std::min(total, s0 + L.T);
            sweep(s0, s1, s0, a->outputs);
            timed(ctx, 1, st, [&] {
                if (ozaki && launch_contract_ozaki<S>((const S *)(ws + L.snap_x), (const S *)(ws + L.snap_y),
                                                      (double *)(ws + L.slot_full), (int)n, L.ld, (int)a->chains,
                                                      a->group_size, s1 - s0, ctx->ozaki.p, ctx->ozaki.bytes, st))
                    return;
                launch_contract<S>((const S *)(ws + L.snap_x), (const S *)(ws + L.snap_y),
                                   (double *)(ws + L.slot_full), (int)n, L.ld, (int)a->chains, a->group_size,
                                   s1 - s0, st);
            });
        }
    }
    if (lerr != cudaSuccess) return fail(ctx, MCINV_E_CUDA, std::string("sweep launch: ") + cudaGetErrorString(lerr));
    CK(cudaGetLastError());
    // moments (the divergence count was produced by the sweep kernels)
    launch_all_moments(ctx, L, ws, a->outputs, nullptr, 0.0, st);
    CK(cudaGetLastError());
    return MCINV_OK;
}

}  // namespace

extern "C" {

const char *mcinv_status_string(mcinv_status st) {
    switch (st) {
        case MCINV_OK: return "ok";
        case MCINV_E_INVALID: return "invalid argument";
        case MCINV_E_ZERO_DIAG: return "zero or missing diagonal element";
        case MCINV_E_DIAG_DOMAIN: return "real path requires a positive diagonal";
        case MCINV_E_DIVERGED: return "chains diverged (sp(T) or sp(S) >= 1)";
        case MCINV_E_NOMEM: return "out of memory";
        case MCINV_E_CUDA: return "CUDA error";
        case MCINV_E_BUFFER: return "buffer too small";
        case MCINV_E_STATE: return "call out of order";
    }
    return "unknown status";
}

mcinv_status mcinv_error_detail(const mcinv_ctx *ctx, int64_t *index, const char **msg) {
    if (!ctx) return MCINV_E_INVALID;
    if (index) *index = ctx->err_index;
    if (msg) *msg = ctx->err.c_str();
    return MCINV_OK;
}

mcinv_status mcinv_create(mcinv_ctx **out, int device, mcinv_dtype dtype, int64_t n, const int64_t *row_ptr,
                          const int32_t *col_idx, const void *values) {
    if (!out) return MCINV_E_INVALID;
    *out = nullptr;
    mcinv_ctx *ctx = new (std::nothrow) mcinv_ctx();
    if (!ctx) return MCINV_E_NOMEM;
    *out = ctx;
    ctx->device = device;
    ctx->dtype = dtype;
    ctx->n = n;
    if (dtype != MCINV_F64 && dtype != MCINV_C128) return fail(ctx, MCINV_E_INVALID, "dtype");
    if (n < 1 || n >= (int64_t(1) << 31)) return fail(ctx, MCINV_E_INVALID, "n out of range");
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, device));
    {
        int l2 = 0;
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device) == cudaSuccess && l2 > 0) ctx->l2_bytes = l2;
    }
    {
        cudaMemPool_t pool;
        uint64_t keep = UINT64_MAX;  // freed blocks stay in the pool: no release to the OS
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess)
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        cudaGetLastError();
    }
    std::vector<std::vector<Entry>> rows;
    TRY(read_csr(ctx, n, row_ptr, col_idx, (const double *)values, dtype == MCINV_C128, rows));
    TRY(dtype == MCINV_C128 ? build_matrix<cd>(ctx, rows) : build_matrix<double>(ctx, rows));
    TRY(default_pattern(ctx));
    CK(cudaStreamSynchronize(0));  // uploads complete before any stream uses them
    ctx->valid = true;
    ctx->err.clear();
    return MCINV_OK;
}

mcinv_status mcinv_set_trace_q(mcinv_ctx *ctx, const int64_t *row_ptr, const int32_t *col_idx, const void *values) {
    if (!ctx || !ctx->valid) return MCINV_E_STATE;
    CK(cudaSetDevice(ctx->device));
    std::vector<std::vector<Entry>> rows;
    TRY(read_csr(ctx, ctx->n, row_ptr, col_idx, (const double *)values, ctx->dtype == MCINV_C128, rows));
    TRY(ctx->dtype == MCINV_C128 ? build_q<cd>(ctx, rows) : build_q<double>(ctx, rows));
    CK(cudaStreamSynchronize(0));
    return MCINV_OK;
}

mcinv_status mcinv_set_pattern(mcinv_ctx *ctx, int64_t count, const int32_t *rows, const int32_t *cols) {
    if (!ctx || !ctx->valid) return MCINV_E_STATE;
    if (count < 0 || count >= (int64_t(1) << 31) || (count > 0 && (!rows || !cols)))
        return fail(ctx, MCINV_E_INVALID, "pattern");
    CK(cudaSetDevice(ctx->device));
    ctx->pattern_custom = true;
    TRY(build_pattern(ctx, count, rows, cols));
    CK(cudaStreamSynchronize(0));
    return MCINV_OK;
}

mcinv_status mcinv_pattern_size(const mcinv_ctx *ctx, int64_t *count) {
    if (!ctx || !ctx->valid || !count) return MCINV_E_STATE;
    *count = ctx->pcount;
    return MCINV_OK;
}

mcinv_status mcinv_workspace_size(const mcinv_ctx *ctx, const mcinv_run_args *args, size_t *bytes) {
    if (!ctx || !ctx->valid || !bytes) return MCINV_E_STATE;
    TRY(check_args(ctx, args));
    *bytes = make_layout(ctx, args).total;
    return MCINV_OK;
}

mcinv_status mcinv_run(mcinv_ctx *ctx, const mcinv_run_args *args) {
    if (!ctx || !ctx->valid) return MCINV_E_STATE;
    TRY(check_args(ctx, args));
    CK(cudaSetDevice(ctx->device));
    const Layout L = make_layout(ctx, args);
    char *ws = (char *)args->workspace;
    if (args->resume) {
        if (!ctx->have_run || ctx->last.chains != args->chains || ctx->last.outputs != args->outputs ||
            ctx->last.group_size != args->group_size || ctx->last.trace_series != args->trace_series ||
            (ws && ws != ctx->ws))
            return fail(ctx, MCINV_E_STATE, "resume needs the previous run's shape and workspace");
    }
    if (ws) {
        if (args->workspace_bytes < L.total || ((uintptr_t)ws & 255))
            return fail(ctx, MCINV_E_BUFFER, "workspace too small or misaligned", (int64_t)L.total);
    } else if (args->resume) {
        // NULL on resume: continue in the previous run's workspace (library-owned or the
        // caller's); the resumed layout is that run's (make_layout keeps its T), so it fits
        if (L.total > ctx->lay.total || L.zw != ctx->lay.zw || L.mom != ctx->lay.mom)
            return fail(ctx, MCINV_E_STATE, "resume layout differs from the previous run's");
        ws = ctx->ws;
    } else {
        if (ctx->own_ws.bytes < L.total) {
            ctx->own_ws.release();
            if (dev_alloc(&ctx->own_ws.p, L.total) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
                cudaGetLastError();
                ctx->own_ws.p = nullptr;
                return fail(ctx, MCINV_E_NOMEM, "workspace allocation", (int64_t)L.total);
            }
            ctx->own_ws.bytes = L.total;
        }
        ws = (char *)ctx->own_ws.p;
    }
    cudaStream_t st = (cudaStream_t)args->stream;
    ctx->have_run = false;
    TRY(ctx->dtype == MCINV_C128 ? run_typed<cd>(ctx, args, L, ws, st) : run_typed<double>(ctx, args, L, ws, st));
    ctx->have_run = true;
    ctx->acc_cycles = args->resume ? ctx->acc_cycles + args->cycles : args->cycles;
    ctx->last = *args;
    ctx->lay = L;
    ctx->ws = ws;
    ctx->stream = st;
    return MCINV_OK;
}

mcinv_status mcinv_accumulators(mcinv_ctx *ctx, double **dev_ptr, size_t *count) {
    if (!ctx || !ctx->have_run || !dev_ptr || !count) return MCINV_E_STATE;
    *dev_ptr = (double *)(ctx->ws + ctx->lay.mom);
    *count = ctx->lay.mom_count;
    return MCINV_OK;
}

mcinv_status mcinv_run_status(mcinv_ctx *ctx, int64_t *diverged) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    CK(cudaSetDevice(ctx->device));
    double bad = 0.0;
    const double *mom = (const double *)(ctx->ws + ctx->lay.mom);
    CK(cudaMemcpyAsync(&bad, mom + ctx->lay.mom_count - 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (diverged) *diverged = (int64_t)bad;
    if (ctx->last_kernel >= 4) {
        unsigned wd = 0;
        CK(cudaMemcpy(&wd, ctx->err_flag.p, sizeof(wd), cudaMemcpyDeviceToHost));
        if (wd) return fail(ctx, MCINV_E_CUDA, "v4 dataflow watchdog: a dependency wait exceeded its bound");
    }
    if (bad > 0.0) return fail(ctx, MCINV_E_DIVERGED, "state non-finite or above 1e12", (int64_t)bad);
    return MCINV_OK;
}

mcinv_status mcinv_recenter(mcinv_ctx *ctx, int64_t total_chains, size_t *m2_offset, size_t *m2_count) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    const mcinv_run_args &a = ctx->last;
    if (total_chains < a.chains || total_chains % a.group_size)
        return fail(ctx, MCINV_E_INVALID, "total_chains");
    CK(cudaSetDevice(ctx->device));
    const Layout &L = ctx->lay;
    const double *s1 = (const double *)(ctx->ws + L.mom);
    launch_all_moments(ctx, L, ctx->ws, a.outputs, s1, (double)(total_chains / a.group_size), ctx->stream);
    CK(cudaGetLastError());
    if (m2_offset) *m2_offset = L.mom_m2;
    if (m2_count) *m2_count = L.mom_m2;
    return MCINV_OK;
}

mcinv_status mcinv_geyer(mcinv_ctx *ctx, double *out) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    if (!out) return fail(ctx, MCINV_E_INVALID, "null out");
    const Layout &L = ctx->lay;
    if (!L.series_cap || ctx->acc_cycles < 1) return fail(ctx, MCINV_E_STATE, "no trace series (trace_series = 0)");
    CK(cudaSetDevice(ctx->device));
    if (ctx->tmp.bytes < 64) {
        ctx->tmp.release();
        if (dev_alloc(&ctx->tmp.p, 64) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
            cudaGetLastError();
            ctx->tmp.p = nullptr;
            return fail(ctx, MCINV_E_NOMEM, "geyer staging");
        }
        ctx->tmp.bytes = 64;
    }
    mcinv::launch_geyer((const double *)(ctx->ws + L.series), ctx->acc_cycles, L.e, (double *)ctx->tmp.p, ctx->stream);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, ctx->tmp.p, 4 * L.e * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return MCINV_OK;
}

mcinv_status mcinv_result(mcinv_ctx *ctx, unsigned output, int64_t total_chains, double *estimate,
                          double *std_error, size_t capacity, int on_device) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    const Layout &L = ctx->lay;
    const mcinv_run_args &a = ctx->last;
    if (!(a.outputs & output) || (output & (output - 1)) || !estimate)
        return fail(ctx, MCINV_E_INVALID, "output not computed by the last run");
    if (total_chains < a.chains || total_chains % a.group_size)
        return fail(ctx, MCINV_E_INVALID, "total_chains");
    if (ctx->acc_cycles < 1)  // burn-in only so far: Eq. (1/C) has no samples to average
        return fail(ctx, MCINV_E_STATE, "no sampling sweeps since the last fresh run (cycles = 0)");
    CK(cudaSetDevice(ctx->device));
    const int64_t n = ctx->n;
    int64_t count = 0;
    size_t off = 0;
    switch (output) {
        case MCINV_DIAG: count = n; off = L.mom_diag; break;
        case MCINV_PATTERN: count = ctx->pcount; off = L.mom_pat; break;
        case MCINV_FULL: count = n * n; off = L.mom_full; break;
        case MCINV_TRACE: count = 1; off = L.mom_trace; break;
        default: return fail(ctx, MCINV_E_INVALID, "output");
    }
    const int64_t comps = count * L.e;
    if (capacity < (size_t)comps) return fail(ctx, MCINV_E_BUFFER, "result buffer too small", comps);
    const double *mom = (const double *)(ctx->ws + L.mom);
    const double cyc = (double)ctx->acc_cycles;  // all sampling sweeps, resumed runs included
    const double G = (double)(total_chains / a.group_size);
    cudaStream_t st = ctx->stream;
    if (on_device) {
        // asynchronous on the run's stream; divergence is reported by mcinv_run_status
        mcinv::launch_finalize(mom + off, mom + off + L.mom_m2, comps, (double)total_chains * cyc, a.group_size * cyc,
                               G, estimate, std_error, st);
        ctx->launches++;
        CK(cudaGetLastError());
        return MCINV_OK;
    }
    const size_t need = 2 * comps * sizeof(double);
    if (ctx->tmp.bytes < need) {
        ctx->tmp.release();
        if (dev_alloc(&ctx->tmp.p, need) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess) {
            cudaGetLastError();
            ctx->tmp.p = nullptr;
            return fail(ctx, MCINV_E_NOMEM, "result staging");
        }
        ctx->tmp.bytes = need;
    }
    double *de = (double *)ctx->tmp.p, *ds = de + comps;
    mcinv::launch_finalize(mom + off, mom + off + L.mom_m2, comps, (double)total_chains * cyc, a.group_size * cyc, G,
                           de, ds, st);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(estimate, de, comps * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (std_error) CK(cudaMemcpyAsync(std_error, ds, comps * sizeof(double), cudaMemcpyDeviceToHost, st));
    return mcinv_run_status(ctx, nullptr);  // synchronizes
}

void mcinv_destroy(mcinv_ctx *ctx) {
    if (!ctx) return;
    if (ctx->valid || ctx->own_ws.p) {
        cudaSetDevice(ctx->device);
        // the buffers are freed stream-ordered on the legacy stream: first let it wait for
        // the last run's stream (a non-blocking caller stream is not ordered with it)
        if (ctx->have_run && ctx->stream) {
            cudaEvent_t ev;
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(ev, ctx->stream);
                cudaStreamWaitEvent(0, ev, 0);
                cudaEventDestroy(ev);
            }
        }
    }
    delete ctx;
}

mcinv_status mcinv_kernel_info(const mcinv_ctx *ctx, int *version, int *chains_per_warp, int64_t *steps_per_sweep) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    if (version) *version = ctx->last_kernel;
    if (chains_per_warp) *chains_per_warp = ctx->last_C;
    if (steps_per_sweep) *steps_per_sweep = ctx->last_steps;
    return MCINV_OK;
}

mcinv_status mcinv_launch_config(const mcinv_ctx *ctx, int *threads, int *chains_per_thread, int *blocks) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    if (threads) *threads = ctx->last_threads;
    if (chains_per_thread) *chains_per_thread = ctx->last_K;
    if (blocks) *blocks = ctx->last_blocks;
    return MCINV_OK;
}

mcinv_status mcinv_set_timing(mcinv_ctx *ctx, int enable) {
    if (!ctx || !ctx->valid) return MCINV_E_STATE;
    ctx->timing = enable != 0;
    return MCINV_OK;
}

mcinv_status mcinv_stats(mcinv_ctx *ctx, int64_t *launches, double *sweep_ms, int64_t *sweep_launches,
                         double *contract_ms, int64_t *contract_launches) {
    if (!ctx || !ctx->valid) return MCINV_E_STATE;
    CK(cudaSetDevice(ctx->device));
    double ms[2] = {0.0, 0.0};
    int64_t cnt[2] = {0, 0};
    for (auto &t : ctx->pending) {
        CK(cudaEventSynchronize(t.b));
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, t.a, t.b));
        ms[t.kind] += f;
        cnt[t.kind]++;
        ctx->event_pool.push_back(t.a);
        ctx->event_pool.push_back(t.b);
    }
    ctx->pending.clear();
    if (launches) *launches = ctx->launches;
    if (sweep_ms) *sweep_ms = ms[0];
    if (sweep_launches) *sweep_launches = cnt[0];
    if (contract_ms) *contract_ms = ms[1];
    if (contract_launches) *contract_launches = cnt[1];
    ctx->launches = 0;
    return MCINV_OK;
}

mcinv_status mcinv_coupled_burn_in(mcinv_ctx *ctx, double tol, int64_t max_sweeps, void *stream, int64_t *sweeps,
                                   double *diff) {
    // Alg. 1 steps 1-5 by Eq. (12): two paths with the same
    // noise differ by a Gauss-Seidel iterate of C d = 0 (z) and C^dagger d = 0 (w),
    // whatever the noise, so the coupled burn-in is the number of noise-free sweeps that
    // take the start difference d0_i = i + 1 (Alg. 1: z_i = 0, z*_i = i, 1-based) below
    // tol in max modulus (reading R23). Runs on one 32-chain group with noise 0.
    if (!ctx || !ctx->valid || !sweeps || !(tol > 0.0) || max_sweeps < 1) return MCINV_E_INVALID;
    CK(cudaSetDevice(ctx->device));
    const int64_t n = ctx->n;
    const int e = ctx->dtype == MCINV_C128 ? 2 : 1;
    mcinv_run_args a{};
    a.seed = 0;
    a.chains = 32;
    a.burn_in = 0;
    a.cycles = 0;
    a.outputs = 0;
    a.noise = MCINV_NOISE_ZERO;
    a.group_size = 32;
    a.stream = stream;
    size_t bytes = 0;
    TRY(mcinv_workspace_size(ctx, &a, &bytes));
    DevBuf tmp;
    if (cudaMalloc(&tmp.p, bytes) != cudaSuccess) {
        cudaGetLastError();
        tmp.p = nullptr;
        return fail(ctx, MCINV_E_NOMEM, "burn-in workspace");
    }
    tmp.bytes = bytes;
    a.workspace = tmp.p;
    a.workspace_bytes = bytes;
    TRY(mcinv_run(ctx, &a));
    std::vector<double> d0((size_t)32 * n * e, 0.0);
    for (int64_t c = 0; c < 32; ++c)
        for (int64_t i = 0; i < n; ++i) d0[(c * n + i) * e] = (double)(i + 1);
    TRY(mcinv_debug_set_state(ctx, 0, 32, d0.data(), d0.data()));
    double *dmax = nullptr;
    CK(cudaMalloc(&dmax, sizeof(double)));
    const Layout L = ctx->lay;
    cudaStream_t st = (cudaStream_t)stream;
    mcinv_status result = MCINV_OK;
    double last = 0.0;
    int64_t p = 0;
    for (p = 1; p <= max_sweeps; ++p) {
        a.resume = 1;
        a.burn_in = 1;
        a.sweep_begin = p - 1;
        result = mcinv_run(ctx, &a);
        if (result != MCINV_OK) break;
        if (ctx->dtype == MCINV_C128)
            mcinv::launch_max_modulus<cd>((const ZW<cd> *)(ctx->ws + L.zw), (int)n, L.ld, dmax, st);
        else
            mcinv::launch_max_modulus<double>((const ZW<double> *)(ctx->ws + L.zw), (int)n, L.ld, dmax, st);
        if (cudaMemcpyAsync(&last, dmax, sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            result = fail(ctx, MCINV_E_CUDA, "burn-in reduction");
            break;
        }
        if (!(last <= 1e12)) {
            result = fail(ctx, MCINV_E_DIVERGED, "coupled paths diverge (sp(T) or sp(S) >= 1)", p);
            break;
        }
        if (last < tol) break;
    }
    cudaFree(dmax);
    ctx->have_run = false;  // the temporary workspace is released
    if (result != MCINV_OK) return result;
    if (diff) *diff = last;
    if (p > max_sweeps) return fail(ctx, MCINV_E_DIVERGED, "burn-in did not reach tol within max_sweeps", max_sweeps);
    *sweeps = p;
    return MCINV_OK;
}

mcinv_status mcinv_run_until(mcinv_ctx *ctx, const mcinv_run_args *args, unsigned output, double rel_se,
                             int64_t check_cycles, int64_t max_cycles, int64_t *cycles_done, double *rel_se_out) {
    // Adaptive stopping (the paper determines M - N "by inserting the
    // calculation of the effective number of cycles during the iteration process"):
    // run args (burn-in included) with check_cycles sampling sweeps, then resume in
    // blocks of check_cycles until max |SE / estimate| of `output` is below rel_se
    // (reading R24; the SE is the group SE of reading R15), or max_cycles.
    if (!ctx || !ctx->valid || !args || !cycles_done || !(rel_se > 0.0) || check_cycles < 1 ||
        max_cycles < check_cycles || !(args->outputs & output) || (output & (output - 1)))
        return MCINV_E_INVALID;
    if (args->chains / args->group_size < 2) return fail(ctx, MCINV_E_INVALID, "run_until needs >= 2 SE groups");
    mcinv_run_args a = *args;
    a.cycles = check_cycles;
    a.resume = 0;
    TRY(mcinv_run(ctx, &a));
    const int64_t count = output == MCINV_DIAG ? ctx->n : output == MCINV_PATTERN ? ctx->pcount
                          : output == MCINV_FULL ? ctx->n * ctx->n : 1;
    const int64_t comps = count * (ctx->dtype == MCINV_C128 ? 2 : 1);
    std::vector<double> est(comps), se(comps);
    int64_t done = check_cycles;
    double worst = 0.0;
    for (;;) {
        TRY(mcinv_result(ctx, output, a.chains, est.data(), se.data(), comps, 0));
        // complex elements: moduli of SE and estimate (the paper's Dirac tolerance is
        // "with respect to the absolute value rather than for real and imaginary part
        // independently")
        worst = 0.0;
        const int e = ctx->dtype == MCINV_C128 ? 2 : 1;
        for (int64_t c = 0; c < count; ++c) {
            const double m = e == 2 ? std::hypot(est[2 * c], est[2 * c + 1]) : std::fabs(est[c]);
            const double s_ = e == 2 ? std::hypot(se[2 * c], se[2 * c + 1]) : se[c];
            worst = std::max(worst, s_ / (m > 0.0 ? m : 1.0));
        }
        if (worst < rel_se || done >= max_cycles) break;
        mcinv_run_args r = a;
        r.resume = 1;
        r.burn_in = 0;
        r.sweep_begin = a.sweep_begin + a.burn_in + done;
        r.cycles = std::min(check_cycles, max_cycles - done);
        TRY(mcinv_run(ctx, &r));
        done += r.cycles;
    }
    *cycles_done = done;
    if (rel_se_out) *rel_se_out = worst;
    return MCINV_OK;
}

mcinv_status mcinv_run_until_geyer(mcinv_ctx *ctx, const mcinv_run_args *args, double rel_se, int64_t check_cycles,
                                   int64_t max_cycles, int64_t *cycles_done, double *rel_se_out) {
    // The paper's stopping rule: after the burn-in, realized traces every
    // cycle; every check_cycles (100 in the paper) the Geyer standard error of their mean
    // relative to the estimate; stop below the tolerance.
    if (!ctx || !ctx->valid || !args || !cycles_done || !(rel_se > 0.0) || check_cycles < 1 ||
        max_cycles < check_cycles || !(args->outputs & MCINV_TRACE))
        return MCINV_E_INVALID;
    mcinv_run_args a = *args;
    a.cycles = check_cycles;
    a.resume = 0;
    a.trace_series = max_cycles;
    TRY(mcinv_run(ctx, &a));
    int64_t done = check_cycles;
    double worst = 0.0;
    const int e = ctx->dtype == MCINV_C128 ? 2 : 1;
    for (;;) {
        double g[8];
        TRY(mcinv_geyer(ctx, g));
        TRY(mcinv_run_status(ctx, nullptr));
        const double mre = g[0], sre = g[2] > 0.0 ? std::sqrt(g[2] / (double)done) : 0.0;
        const double mim = e == 2 ? g[4] : 0.0, sim = (e == 2 && g[6] > 0.0) ? std::sqrt(g[6] / (double)done) : 0.0;
        const double m = std::hypot(mre, mim), se = std::hypot(sre, sim);
        worst = se / (m > 0.0 ? m : 1.0);
        if (worst < rel_se || done >= max_cycles) break;
        mcinv_run_args r = a;
        r.resume = 1;
        r.burn_in = 0;
        r.sweep_begin = a.sweep_begin + a.burn_in + done;
        r.cycles = std::min(check_cycles, max_cycles - done);
        TRY(mcinv_run(ctx, &r));
        done += r.cycles;
    }
    *cycles_done = done;
    if (rel_se_out) *rel_se_out = worst;
    return MCINV_OK;
}

mcinv_status mcinv_debug_levels(mcinv_dtype dtype, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                const void *values, const int64_t *q_row_ptr, const int32_t *q_col_idx,
                                const void *q_values, unsigned outputs, int32_t *level, int64_t *info,
                                int slot_R, int slot_L, int32_t *info_slots, int64_t slots_capacity) {
    if (!info) return MCINV_E_INVALID;
    mcinv_ctx c;
    mcinv_ctx *ctx = &c;
    ctx->host_only = true;
    ctx->dtype = dtype;
    ctx->n = n;
    if (dtype != MCINV_F64 && dtype != MCINV_C128) return MCINV_E_INVALID;
    if (n < 1 || n >= (int64_t(1) << 31)) return MCINV_E_INVALID;
    std::vector<std::vector<Entry>> rows;
    TRY(read_csr(ctx, n, row_ptr, col_idx, (const double *)values, dtype == MCINV_C128, rows));
    TRY(dtype == MCINV_C128 ? build_matrix<cd>(ctx, rows) : build_matrix<double>(ctx, rows));
    TRY(default_pattern(ctx));
    if (q_row_ptr) {
        std::vector<std::vector<Entry>> qrows;
        TRY(read_csr(ctx, n, q_row_ptr, q_col_idx, (const double *)q_values, dtype == MCINV_C128, qrows));
        TRY(dtype == MCINV_C128 ? build_q<cd>(ctx, qrows) : build_q<double>(ctx, qrows));
    }
    LevelDev *lv = dtype == MCINV_C128 ? get_levels<cd>(ctx, outputs) : get_levels<double>(ctx, outputs);
    if (!lv->error.empty()) return fail(ctx, MCINV_E_INVALID, lv->error);
    const mcinv::LevelPlan &P = lv->host;
    if (info_slots) {
        // v4 slot schedule of this plan for R rows per warp group and slack L (levels.h)
        std::vector<int4> rec(n);
        for (int64_t o = 0; o < n; ++o) {
            const int i = P.ord_row[o], beg = P.ord_eptr[o], cnt = P.ord_eptr[o + 1] - beg;
            int nlow = 0;
            while (nlow < cnt && P.ent_col[beg + nlow] < i) ++nlow;
            if (cnt >= 65536) return fail(ctx, MCINV_E_INVALID, "a row has 65536 or more off-diagonal entries", i);
            rec[o] = make_int4(i, beg, (int)((unsigned)cnt | (unsigned)nlow << 16), -1);
        }
        const char *se = std::getenv("MCINV_SIMILAR");
        const std::vector<int> order = mcinv::schedule_slots(n, rec, P.ent_col, slot_R, slot_L, 0, se ? std::atoi(se) : 64);
        if ((int64_t)order.size() > slots_capacity) return fail(ctx, MCINV_E_BUFFER, "slots", (int64_t)order.size());
        for (size_t t = 0; t < order.size(); ++t) info_slots[t] = order[t] < 0 ? -1 : P.ord_row[order[t]];
        info[6] = (int64_t)order.size();
    }
    info[0] = P.D;
    info[1] = P.max_rows;
    info[2] = P.fused_pairs;
    info[3] = P.deferred_pairs;
    info[4] = (int64_t)P.tq_row.size();
    info[5] = (int64_t)P.ent_col.size() - 8;  // without the kernel padding
    if (level) std::copy(P.level.begin(), P.level.end(), level);
    return MCINV_OK;
}

mcinv_status mcinv_debug_blocks(mcinv_dtype dtype, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                const void *values, const int64_t *q_row_ptr, const int32_t *q_col_idx,
                                const void *q_values, unsigned outputs, int R, int W, int pad_ku, int ecap, int wmask,
                                int32_t *slot_x, uint32_t *masks, int64_t capacity, int64_t *nslots) {
    if (!nslots || R < 1 || 32 % R || W < 1) return MCINV_E_INVALID;
    mcinv_ctx c;
    mcinv_ctx *ctx = &c;
    ctx->host_only = true;
    ctx->dtype = dtype;
    ctx->n = n;
    if (dtype != MCINV_F64 && dtype != MCINV_C128) return MCINV_E_INVALID;
    if (n < 1 || n >= (int64_t(1) << 31)) return MCINV_E_INVALID;
    std::vector<std::vector<Entry>> rows;
    TRY(read_csr(ctx, n, row_ptr, col_idx, (const double *)values, dtype == MCINV_C128, rows));
    TRY(dtype == MCINV_C128 ? build_matrix<cd>(ctx, rows) : build_matrix<double>(ctx, rows));
    TRY(default_pattern(ctx));
    if (q_row_ptr) {
        std::vector<std::vector<Entry>> qrows;
        TRY(read_csr(ctx, n, q_row_ptr, q_col_idx, (const double *)q_values, dtype == MCINV_C128, qrows));
        TRY(dtype == MCINV_C128 ? build_q<cd>(ctx, qrows) : build_q<double>(ctx, qrows));
    }
    LevelDev *lv = dtype == MCINV_C128 ? get_levels<cd>(ctx, outputs) : get_levels<double>(ctx, outputs);
    if (!lv->error.empty()) return fail(ctx, MCINV_E_INVALID, lv->error);
    LevelDev::Slots *sl = dtype == MCINV_C128 ? get_slots<cd>(ctx, lv, R, W, true, pad_ku, ecap, wmask != 0)
                                               : get_slots<double>(ctx, lv, R, W, true, pad_ku, ecap, wmask != 0);
    if (!sl) return fail(ctx, MCINV_E_INVALID, "slot schedule");
    *nslots = (int64_t)sl->h_x.size();
    if (*nslots > capacity) return fail(ctx, MCINV_E_BUFFER, "slots", *nslots);
    if (slot_x) std::copy(sl->h_x.begin(), sl->h_x.end(), slot_x);
    if (masks) std::copy(sl->h_mask.begin(), sl->h_mask.end(), masks);
    return MCINV_OK;
}

mcinv_status mcinv_debug_philox(int device, uint64_t seed, int64_t count, const uint32_t *ctr4, uint32_t *out4) {
    mcinv_ctx *ctx = nullptr;
    if (count < 0 || (count > 0 && (!ctr4 || !out4))) return MCINV_E_INVALID;
    if (count == 0) return MCINV_OK;
    CK(cudaSetDevice(device));
    uint32_t *dc = nullptr, *dout = nullptr;
    CK(cudaMalloc(&dc, count * 16));
    CK(cudaMalloc(&dout, count * 16));
    CK(cudaMemcpy(dc, ctr4, count * 16, cudaMemcpyHostToDevice));
    mcinv::launch_philox(dc, count, (uint32_t)seed, (uint32_t)(seed >> 32), dout, nullptr, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out4, dout, count * 16, cudaMemcpyDeviceToHost));
    cudaFree(dc);
    cudaFree(dout);
    return MCINV_OK;
}

mcinv_status mcinv_debug_gaussian(int device, uint64_t seed, int64_t count, const uint32_t *ctr4, double *out) {
    mcinv_ctx *ctx = nullptr;
    if (count < 0 || (count > 0 && (!ctr4 || !out))) return MCINV_E_INVALID;
    if (count == 0) return MCINV_OK;
    CK(cudaSetDevice(device));
    uint32_t *dc = nullptr;
    double *dout = nullptr;
    CK(cudaMalloc(&dc, count * 16));
    CK(cudaMalloc(&dout, count * 8));
    CK(cudaMemcpy(dc, ctr4, count * 16, cudaMemcpyHostToDevice));
    mcinv::launch_philox(dc, count, (uint32_t)seed, (uint32_t)(seed >> 32), nullptr, dout, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, dout, count * 8, cudaMemcpyDeviceToHost));
    cudaFree(dc);
    cudaFree(dout);
    return MCINV_OK;
}

static mcinv_status state_io(mcinv_ctx *ctx, int64_t chain_begin, int64_t chains, void *z, void *w, bool get) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    if (chain_begin < 0 || chains < 0 || chain_begin + chains > ctx->last.chains || !z || !w)
        return fail(ctx, MCINV_E_INVALID, "state range");
    if (chains == 0) return MCINV_OK;
    CK(cudaSetDevice(ctx->device));
    const int64_t n = ctx->n, ld = ctx->lay.ld, e = ctx->lay.e;
    // only the requested chains cross the bus: one strided 2-D copy of n rows of `chains`
    // contiguous (z, w) elements (config 4: 3 chains x 1e6 rows = 48 MB, not the 131 GB state)
    const size_t elem = 2 * (size_t)e * sizeof(double);  // one ZW<S>
    std::vector<double> buf((size_t)n * chains * 2 * e);
    char *dev = ctx->ws + ctx->lay.zw + (size_t)chain_begin * elem;
    CK(cudaStreamSynchronize(ctx->stream));
    if (get)
        CK(cudaMemcpy2D(buf.data(), chains * elem, dev, ld * elem, chains * elem, n, cudaMemcpyDeviceToHost));
    double *zd = (double *)z, *wd = (double *)w;
    for (int64_t c = 0; c < chains; ++c)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t q = 0; q < e; ++q) {
                double *src = &buf[((i * chains + c) * 2) * e + q];
                double *hz = &zd[(c * n + i) * e + q], *hw = &wd[(c * n + i) * e + q];
                if (get) {
                    *hz = src[0];
                    *hw = src[e];
                } else {
                    src[0] = *hz;
                    src[e] = *hw;
                }
            }
    if (!get)
        CK(cudaMemcpy2D(dev, ld * elem, buf.data(), chains * elem, chains * elem, n, cudaMemcpyHostToDevice));
    return MCINV_OK;
}

mcinv_status mcinv_debug_group_sums(mcinv_ctx *ctx, unsigned output, int64_t group_begin, int64_t groups,
                                    double *out) {
    if (!ctx || !ctx->have_run) return MCINV_E_STATE;
    const Layout &L = ctx->lay;
    const mcinv_run_args &a = ctx->last;
    if (!(a.outputs & output) || (output & (output - 1)) || !out || group_begin < 0 || groups < 0 ||
        group_begin + groups > L.G)
        return fail(ctx, MCINV_E_INVALID, "group range or output");
    CK(cudaSetDevice(ctx->device));
    int64_t count = 0;
    size_t slot = 0;
    switch (output) {
        case MCINV_DIAG: count = ctx->n; slot = L.slot_diag; break;
        case MCINV_PATTERN: count = ctx->pcount; slot = L.slot_pat; break;
        case MCINV_FULL: count = ctx->n * ctx->n; slot = L.slot_full; break;
        default: count = 1; slot = L.slot_trace; break;
    }
    const size_t row = (size_t)count * L.e * sizeof(double);  // one group's accumulators (ksub == 1)
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(out, ctx->ws + slot + (size_t)group_begin * row, (size_t)groups * row, cudaMemcpyDeviceToHost));
    return MCINV_OK;
}

mcinv_status mcinv_debug_get_state(mcinv_ctx *ctx, int64_t chain_begin, int64_t chains, void *z, void *w) {
    return state_io(ctx, chain_begin, chains, z, w, true);
}

mcinv_status mcinv_debug_set_state(mcinv_ctx *ctx, int64_t chain_begin, int64_t chains, const void *z,
                                   const void *w) {
    return state_io(ctx, chain_begin, chains, const_cast<void *>(z), const_cast<void *>(w), false);
}

}  // extern "C"
