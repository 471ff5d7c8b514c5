// mcinv_internal.cuh -- types shared by the host library (mcinv_host.cu) and
// the device kernels (sweep.cu, contract.cu, reduce.cu). Product code only;
// nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// v5 gather unroll (entries in flight per thread): real / complex; the host pads every row's
// block entries to a multiple of it
#ifndef MCINV_V5_KUR
#define MCINV_V5_KUR 4
#endif
#ifndef MCINV_V5_KUC
#define MCINV_V5_KUC 2
#endif

namespace mcinv {

// Complex double, interleaved (re, im) as in the ABI.
struct __align__(16) cd {
    double re, im;
};

// One (row, chain) state element: z_i and w_i of Eq. (4)/(5) side by side,
// so that one coalesced load serves both updates when row i and column i of
// C share their pattern (every BASELINE config).
template <typename S> struct __align__(2 * sizeof(S)) ZW {
    S z, w;
};

// Device copy of C (built by mcinv_create):
//  u_ptr/u_col: per row i the sorted UNION of {j : c_ij != 0} and
//               {j : c_ji != 0}, j != i (structural, explicit zeros kept);
//  u_a[e] = c_ij        (0 if absent)  -> Eq. (4) term
//  u_b[e] = conj(c_ji)  (0 if absent)  -> Eq. (5) term
//  delta = 1/c_ii, sigma = 1/sqrt(c_ii) (principal branch).
template <typename S> struct DevMatrix {
    int n;
    const int *u_ptr;
    const int *u_col;
    const S *u_a;
    const S *u_b;
    const S *delta;
    const S *sigma;
};

// Pattern lists, by the row r = max(i, j) at which both z_i and w_j are
// final within a sweep: p_other encodes the partner index and, in bit 31,
// which side is the current row (0: z_r conj(w_other); 1: z_other conj(w_r)).
struct DevPattern {
    int count;
    const int *p_ptr;
    const int *p_idx;
    const int *p_other;
};

// Q lists of the trace w^dagger Q z split by r = max(i, j):
//  row part  qr: entries (j, Q_rj), j <= r   -> conj(w_r) * sum Q_rj z_j
//  col part  qc: entries (i, Q_ir), i <  r   -> z_r * sum Q_ir conj(w_i)
template <typename S> struct DevQ {
    const int *qr_ptr;
    const int *qr_col;
    const S *qr_val;
    const int *qc_ptr;
    const int *qc_row;
    const S *qc_val;
};

enum : unsigned { OUT_DIAG = 1u, OUT_PATTERN = 2u, OUT_FULL = 4u, OUT_TRACE = 8u };

template <typename S> struct SweepParams {
    DevMatrix<S> A;
    DevPattern P;
    DevQ<S> Q;
    ZW<S> *zw;          // [n][ld]
    int ld;             // chains padded to a multiple of 32
    int chains;         // active chains
    uint32_t chain0;    // global index of local chain 0
    uint32_t key0, key1;
    int noise;
    uint32_t sweep_abs0;  // absolute sweep index of local sweep 0
    int s_begin, s_end;   // local sweep range of this launch
    int burn_in;
    unsigned outputs;
    int gs;               // group size
    int G;                // groups in this run
    double *slot_diag;    // [G][n] * e
    double *slot_pat;     // [G][pcount] * e
    double *slot_trace;   // [G] * e
    S *snap_x, *snap_y;   // [T][n][ld]
    int snap_s0;          // local sweep stored at snapshot slot 0
    double *bad;          // divergence count (+1 per active lane that stored a value above 1e12 or non-finite)
    double *series;       // TRACE: per sampling sweep, the run's summed w^dagger Q z (Geyer's series), or null
    int series_base;      // series index of this launch's first sampling sweep
};

template <typename S>
void launch_sweep(const SweepParams<S> &p, cudaStream_t st);

// v3 sweep kernel on the level schedule (levels.h / sweep3.cu). Arrays are in
// level order; see LevelPlan for their meaning.
template <typename S>
struct Sweep3Params {
    const int *ph_row;
    const int4 *ord_rec;  // [n] level-order row records {i, entry begin, entries | lower entries << 16,
                          //     pattern slot of (i,i) or -1}
    const int *ent_col;
    const S *ent_ab;      // [nnz_u][2]: a = c_ij (Eq. 4), b = conj(c_ji) (Eq. 5)
    const int2 *ent_pz;   // [nnz_u] pattern slots, or nullptr
    const S *ord_dsg;     // [n][2]: delta_i, sigma_i
    const int *ph_tq, *tq_row, *tq_eptr, *tq_col;
    const S *tq_val;
    const int *ph_pp, *pp_i, *pp_j, *pp_slot;
    int D;
    ZW<S> *zw;
    int n, ld, chains;
    uint32_t chain0, key0, key1;
    int noise;
    uint32_t sweep_abs0;
    int s_begin, s_end, burn_in;
    unsigned outputs;
    int lgC;              // log2 chains per CTA
    int lgP;              // log2 lanes of one SE group inside a CTA: min(group size, C) / K (kernel template)
    int lgG;              // log2 group size: chain c accumulates into group slot c >> lgG
    int lgK;              // v3: log2 chains per thread (1 only for real runs without trace / deferred items)
    int pcount;
    double *slot_diag, *slot_pat, *slot_trace;  // [groups][count] (x e doubles)
    S *snap_x, *snap_y;
    int snap_s0;
    // v4 (dataflow) only: level-order rows padded per level to whole warp groups of
    // R = 32 / C rows; slot_rec.x = -1 marks padding
    const int4 *slot_rec;
    const S *slot_dsg;
    int nslots;
    unsigned *err;        // set (watchdog) if a dependency wait exceeds its bound
    // v5 (v4 + TMA-staged plan): per warp group one contiguous block (see get_slots)
    const unsigned char *blob;
    const int64_t *gofs;  // [groups + 1] byte offsets of the blocks in blob
    int maxb;             // largest block (bytes)
    int spin_ns;          // dataflow waits: __nanosleep between counter polls (0: none)
    int reconv;           // v5: __syncwarp at the item end (bit 0) / after the dependency waits (bit 1)
    int prefetch;         // v5: prefetch upper neighbours' lines before the noise (0 off, 1 L1, 2 L2)
    double *bad;          // divergence count: +1 per active lane that stored a non-finite value or one
                          // above 1e12 in modulus (checked at every update = every sweep's end state)
    double *series;       // TRACE: per sampling sweep, the run's summed w^dagger Q z (Geyer's series), or null
    int series_base;      // series index of this launch's first sampling sweep
};

template <typename S>
cudaError_t launch_sweep3(const Sweep3Params<S> &p, int threads, cudaStream_t st);
// v4: per-row completion counters in shared memory instead of per-level barriers
template <typename S>
cudaError_t launch_sweep4(const Sweep3Params<S> &p, int threads, cudaStream_t st);
// v5: v4 with each warp group's plan data staged into shared memory by TMA bulk copies
template <typename S>
cudaError_t launch_sweep5(const Sweep3Params<S> &p, int threads, cudaStream_t st);
size_t sweep5_smem(int n, int threads, int maxb);
constexpr int kByteCounters = 160000;  // dataflow kernels: above, one completion bit per row in shared memory
// v6: v5 with two chains per thread (real C; the chain pair shares one Box-Muller pair)
cudaError_t launch_sweep6(const Sweep3Params<double> &p, int threads, cudaStream_t st);
int sweep6_ku(int threads);
size_t sweep6_smem(int n, int threads, int maxb);  // two block slots per warp  // v6's gather unroll for a thread count (the blocks' entry padding)

// A_g[i][j] += sum_{t < T, c in group g} X[t][i][c] conj(Y[t][j][c]).
template <typename S>
void launch_contract(const S *x, const S *y, double *acc, int n, int ld, int chains, int gs, int T,
                     cudaStream_t st);

// K3 by the Ozaki scheme on tcgen05 int8 (contract_ozaki.cu): scratch bytes for an n x K chunk,
// and the launch (false: not applicable, the DMMA kernel runs instead)
size_t contract_ozaki_scratch(int n, int K, bool cplx, int groups);
template <typename S>
bool launch_contract_ozaki(const S *x, const S *y, double *acc, int n, int ld, int chains, int gs, int T,
                           void *scratch, size_t scratch_bytes, cudaStream_t st);

// slot layout [G * k][comps]: group g is the sum of sub-slots g*k .. g*k+k-1
// s1 = sum of the group sums, m2 = their scatter about the mean of these groups (center ==
// nullptr) or about center[c] / center_G (the global mean after an all-reduce; s1 untouched)
void launch_moments(const double *slot, int G, int k, int64_t comps, double *s1, double *m2, const double *center,
                    double center_G, cudaStream_t st);
void launch_finalize(const double *s1, const double *m2, int64_t comps, double m_cycles, double gs_cycles,
                     double G, double *est, double *se, cudaStream_t st);
template <typename S>
void launch_max_modulus(const ZW<S> *zw, int n, int ld, double *out, cudaStream_t st);
// Geyer's initial positive sequence estimator of each component of a series x[m][e]:
// out[c * 4 + {0..3}] = {mean, gamma_0, sigma2 = m Var(mean), effective length}
void launch_geyer(const double *x, int64_t m, int e, double *out, cudaStream_t st);
void launch_philox(const uint32_t *ctr, int64_t count, uint32_t k0, uint32_t k1, uint32_t *out,
                   double *gauss, cudaStream_t st);

}  // namespace mcinv
