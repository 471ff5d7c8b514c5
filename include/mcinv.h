/*
 * mcinv.h -- C99 ABI of the B200-native correlated-chains (CC) Monte Carlo
 * matrix inverter (Garcia-Cortes & Cabrillo, arXiv cs/0412107).
 *
 * The method (PAPER.md, "P:<line>"): many independent chains each update two
 * coupled vectors z and w row by row in Gauss-Seidel order with a shared
 * noise draw phi (Eq. 4 and Eq. 5; Eq. 5a/5b). After a
 * burn-in of N sweeps the products z w^dagger average to C^-1 (Eq. 1/C,
 * P:173-176), and w^dagger Q z to tr(Q C^-1) (Eq. tr; see
 * DESIGN.md reading R2 for the conjugation). This library estimates, for a
 * sparse real (f64) or complex (c128) C given in CSR form:
 *   MCINV_DIAG    diag(C^-1)                     (n values)
 *   MCINV_PATTERN selected elements (C^-1)_{ij}  (default: the pattern of C)
 *   MCINV_FULL    the dense C^-1                 (n*n values, row-major)
 *   MCINV_TRACE   tr(Q C^-1) for a sparse Q      (1 value)
 * each with a Monte Carlo standard error from disjoint chain groups.
 *
 * Conventions
 *  - Every call returns mcinv_status; no C++ exception crosses the ABI.
 *  - Indices are 0-based. CSR: row_ptr[0] = 0, non-decreasing, row_ptr[n] =
 *    nnz; col_idx in [0, n). Duplicates are summed; explicit zeros are kept.
 *  - c128 values are interleaved double pairs (re, im); estimates and standard
 *    errors of complex outputs are interleaved too (the standard error pair
 *    holds the SE of the real and of the imaginary part).
 *  - Host inputs are copied during the call; the caller may free them on
 *    return. All device memory of C and Q is owned by the context.
 *  - The hot path (mcinv_run) is asynchronous on the caller's CUDA stream.
 *  - Thread safety: one context per host thread and stream.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one returns MCINV_E_CUDA.
 */
#ifndef MCINV_H
#define MCINV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mcinv_ctx mcinv_ctx;   /* opaque; owns device copies of C and Q */

typedef enum {
    MCINV_OK = 0,
    MCINV_E_INVALID = 1,      /* bad argument, bad CSR, non-finite value */
    MCINV_E_ZERO_DIAG = 2,    /* missing or zero c_ii: D must be non-singular */
    MCINV_E_DIAG_DOMAIN = 3,  /* real path with c_ii <= 0 (1/sqrt(c_ii) not real; use C128) */
    MCINV_E_DIVERGED = 4,     /* non-finite or |z|,|w| > 1e12 after any sweep: sp(T) or sp(S) >= 1 */
    MCINV_E_NOMEM = 5,        /* device or host allocation failed */
    MCINV_E_CUDA = 6,         /* CUDA runtime error (message via mcinv_error_detail) */
    MCINV_E_BUFFER = 7,       /* caller buffer too small; required size via mcinv_error_detail */
    MCINV_E_STATE = 8         /* call out of order (e.g. result before run, resume without state) */
} mcinv_status;

typedef enum { MCINV_F64 = 1, MCINV_C128 = 2 } mcinv_dtype;

enum { MCINV_DIAG = 1u, MCINV_PATTERN = 2u, MCINV_FULL = 4u, MCINV_TRACE = 8u };

/* Noise source for Eq. (4)/(5): Gaussian (BASELINE north_star; DESIGN.md
 * reading R4), Z2 = +-1 (the paper's preferred bounded noise phi = 2B - 1,
 * P:123-126; reading R21), or the constants 0 and 1 (test modes: zero
 * noise reduces CC to Gauss-Seidel, Eq. 12). */
enum { MCINV_NOISE_GAUSS = 0, MCINV_NOISE_ZERO = 1, MCINV_NOISE_ONE = 2, MCINV_NOISE_Z2 = 3 };

/* Build a context for C on CUDA device `device`: validates the CSR, splits
 * C = L + D + U, builds the row lists of Eq. (4) and the
 * conjugated column lists of Eq. (5), 1/c_ii and 1/sqrt(c_ii) (principal
 * branch; Eq. 5 uses their conjugates, reading R1), and uploads
 * them. values: nnz doubles (F64) or 2*nnz doubles (C128).
 * Errors: E_INVALID, E_ZERO_DIAG, E_DIAG_DOMAIN, E_NOMEM, E_CUDA. On any
 * error *out receives a context that holds only the error detail (offending
 * row via mcinv_error_detail); it must still be destroyed. */
mcinv_status mcinv_create(mcinv_ctx **out, int device, mcinv_dtype dtype, int64_t n,
                          const int64_t *row_ptr, const int32_t *col_idx, const void *values);

/* Weighting matrix Q of Eq. (tr), same dtype and order as C.
 * Needed for MCINV_TRACE. The estimator is w^dagger Q z (reading R2). */
mcinv_status mcinv_set_trace_q(mcinv_ctx *ctx, const int64_t *row_ptr, const int32_t *col_idx,
                               const void *values);

/* Elements (rows[p], cols[p]) of C^-1 estimated by MCINV_PATTERN, in this
 * order. Default (never called): the structural pattern of C in CSR order,
 * diagonal included. */
mcinv_status mcinv_set_pattern(mcinv_ctx *ctx, int64_t count, const int32_t *rows, const int32_t *cols);

/* Number of pattern elements currently configured (for sizing results). */
mcinv_status mcinv_pattern_size(const mcinv_ctx *ctx, int64_t *count);

typedef struct {
    uint64_t seed;          /* Philox key (noise phi(c,k,i) keyed by (seed, chain, sweep, row)) */
    int64_t chain_begin;    /* global index of the first chain of this call (multiple of group_size) */
    int64_t chains;         /* chains in this call (multiple of group_size, >= 1) */
    int64_t burn_in;        /* N: sweeps discarded */
    int64_t cycles;         /* M - N: sampling sweeps accumulated */
    int64_t sweep_begin;    /* absolute index of the first sweep (resume keeps the noise stream) */
    unsigned outputs;       /* OR of MCINV_DIAG | MCINV_PATTERN | MCINV_FULL | MCINV_TRACE */
    int noise;              /* MCINV_NOISE_* */
    int group_size;         /* chains per standard-error group: 1, 2, 4, 8, 16 or 32 */
    int resume;             /* 0: z = w = 0 (Alg. 1 step 1), accumulators zeroed;
                               1: continue from the state and accumulators in `workspace` */
    int snapshot_sweeps;    /* MCINV_FULL: sweeps per X Y^dagger contraction chunk (0 = auto) */
    void *workspace;        /* device memory of >= mcinv_workspace_size bytes, 256-B aligned, or
                               NULL to let the library allocate (and own) it */
    size_t workspace_bytes;
    void *stream;           /* cudaStream_t; NULL = legacy default stream */
    int64_t trace_series;   /* MCINV_TRACE: capacity (sampling sweeps since the fresh run) of the
                               series of realized traces, one per sampling sweep summed over the
                               run's chains, for Geyer's effective length (mcinv_geyer); 0 = off.
                               A resumed run must pass the capacity of the run it continues. */
} mcinv_run_args;

/* Device workspace needed by mcinv_run with these arguments (state Z/W,
 * per-group accumulators, contraction snapshots, moments). */
mcinv_status mcinv_workspace_size(const mcinv_ctx *ctx, const mcinv_run_args *args, size_t *bytes);

/* Run chains [chain_begin, chain_begin + chains) for burn_in + cycles sweeps
 * (Alg. 1 with a fixed burn-in), asynchronously on args->stream.
 * On return the per-output moment vectors (see mcinv_accumulators) are being
 * produced on the stream. Errors detected on the device (divergence) are
 * reported by mcinv_result. */
mcinv_status mcinv_run(mcinv_ctx *ctx, const mcinv_run_args *args);

/* Coupled burn-in (Alg. 1 steps 1-5; NEXT-2): the number of sweeps
 * after which two paths started at z = w = 0 and z*_i = w*_i = i (1-based) and
 * driven by the same noise agree to `tol` in max modulus over all rows of z and
 * w (reading R23). By Eq. (12) their difference is a noise-free
 * Gauss-Seidel iterate of C d = 0 and C^dagger d = 0, so it is computed on one
 * noise-free path from d0 (exact, and the same for every chain). *sweeps
 * receives that count (use it as burn_in), *diff (may be NULL) the final max
 * difference. Uses a temporary workspace and replaces the context's last-run
 * state (call before mcinv_run). Synchronizes `stream`. Errors: E_INVALID (tol
 * <= 0, max_sweeps < 1), E_DIVERGED (difference non-finite or above 1e12, or
 * tol not reached within max_sweeps: sp(T) or sp(S) >= 1). */
mcinv_status mcinv_coupled_burn_in(mcinv_ctx *ctx, double tol, int64_t max_sweeps, void *stream, int64_t *sweeps,
                                   double *diff);

/* Adaptive stopping (NEXT-2; the paper determines M - N during the run,
 * P:359-377, Tables 2/4/5): run `args` (burn_in included, args->cycles
 * ignored) with check_cycles sampling sweeps, then resume in blocks of
 * check_cycles until max over the elements of |SE| / |estimate| (moduli for
 * complex elements) of `output` (one
 * MCINV_* bit present in args->outputs) is below rel_se, or max_cycles sampling
 * sweeps are done (reading R24). *cycles_done receives the sampling sweeps run,
 * *rel_se_out (may be NULL) the final relative SE. Needs >= 2 SE groups.
 * Synchronizes; mcinv_result then reads the final estimate. */
mcinv_status mcinv_run_until(mcinv_ctx *ctx, const mcinv_run_args *args, unsigned output, double rel_se,
                             int64_t check_cycles, int64_t max_cycles, int64_t *cycles_done, double *rel_se_out);

/* Geyer's effective sample size of the trace (the paper's standard
 * errors): from the series of realized traces w^dagger Q z, one value per
 * sampling sweep since the last fresh run summed over the run's chains (a run
 * with MCINV_TRACE and trace_series > 0), Geyer's initial positive sequence
 * estimator gives per component (re; and im for C128) out[4c .. 4c+3] =
 * {series mean, gamma_0, sigma2 = M Var(series mean), effective length
 * M gamma_0 / sigma2}, M = the sampling sweeps so far. The trace estimate is
 * mean / chains with Geyer standard error sqrt(sigma2 / M) / chains.
 * Synchronizes. Errors: E_STATE (no series: TRACE with trace_series = 0, or no
 * sampling sweep yet), E_INVALID (null out). */
mcinv_status mcinv_geyer(mcinv_ctx *ctx, double *out);

/* Adaptive stopping with the paper's rule: run `args` (burn_in
 * included, args->cycles ignored, TRACE required) and resume in blocks of
 * check_cycles (the paper: 100) until the trace's Geyer relative standard
 * error |SE| / |estimate| (moduli for complex; SE from mcinv_geyer)
 * is below rel_se, or max_cycles sampling sweeps are done. *cycles_done and
 * *rel_se_out (may be NULL) receive the sweeps run and the final relative SE.
 * The series capacity is max_cycles. Synchronizes. */
mcinv_status mcinv_run_until_geyer(mcinv_ctx *ctx, const mcinv_run_args *args, double rel_se, int64_t check_cycles,
                                   int64_t max_cycles, int64_t *cycles_done, double *rel_se_out);

/* Borrowed device pointer to the moment vector of the last run, for an
 * all-reduce (SUM, float64) across GPUs that ran disjoint chain ranges:
 *   S1 of each output present, in the order DIAG, PATTERN, FULL, TRACE
 *       (count*e doubles each; e = 1 real, 2 complex: re and im parts),
 *   then M2 of each output in the same order (the same sizes),
 *   then one double: the divergence count (non-zero if any chain diverged).
 * S1 = sum over this run's SE groups of the group sums (Eq. 1/C numerator);
 * M2 = sum of the squared deviations of the group sums from their mean, taken
 * two-pass about the mean of THIS run's groups (no raw sum of squares: no
 * cancellation). On one GPU the vector is final. Across GPUs: SUM-all-reduce
 * the whole vector, call mcinv_recenter (M2 about the global mean), then
 * SUM-all-reduce the M2 block it reports. Valid until the next run or destroy. */
mcinv_status mcinv_accumulators(mcinv_ctx *ctx, double **dev_ptr, size_t *count);

/* After a SUM all-reduce of the moment vector across the ranks of one job:
 * recompute this rank's M2 block about the global mean S1 / G_total (G_total =
 * total_chains / group_size) from its resident group sums, so that a second SUM
 * all-reduce of the M2 block (doubles [*m2_offset, *m2_offset + *m2_count) of
 * the vector) gives the scatter of all groups about the global mean.
 * Asynchronous on the run's stream. Errors: E_STATE (no run), E_INVALID
 * (total_chains smaller than this run or not a multiple of group_size). */
mcinv_status mcinv_recenter(mcinv_ctx *ctx, int64_t total_chains, size_t *m2_offset, size_t *m2_count);

/* Synchronize the last run's stream and report its device-side status:
 * E_DIVERGED if any chain stored a non-finite value or one above 1e12 in
 * modulus after any sweep (reading R12; *diverged, may be NULL, receives the
 * count of affected chains x launches), E_CUDA if a dataflow dependency wait
 * timed out (watchdog), else OK. */
mcinv_status mcinv_run_status(mcinv_ctx *ctx, int64_t *diverged);

/* Estimate and standard error of one output from the (possibly all-reduced)
 * moments: estimate = S1 / (total_chains * cycles) (Eq. 1/C), cycles =
 * all sampling sweeps since the last non-resume run; SE =
 * sd(group means)/sqrt(G) = sqrt(M2 / (G - 1) / G) / (group_size * cycles),
 * G = total_chains / group_size (R15; NaN for G = 1).
 * estimate / std_error receive count*e doubles each (std_error may be NULL);
 * capacity is in doubles. on_device != 0: both are device pointers, written
 * asynchronously on the run's stream with no host synchronization (check the
 * run with mcinv_run_status); otherwise host pointers, and the call
 * synchronizes and returns mcinv_run_status's verdict (E_DIVERGED, E_CUDA).
 * E_BUFFER (required capacity via mcinv_error_detail's index) if capacity is
 * too small, E_STATE if no sampling sweep has run since the last fresh run
 * (cycles = 0: a burn-in-only run, to be continued with resume = 1). */
mcinv_status mcinv_result(mcinv_ctx *ctx, unsigned output, int64_t total_chains,
                          double *estimate, double *std_error, size_t capacity, int on_device);

const char *mcinv_status_string(mcinv_status st);

/* Last error of this context: index (row, required capacity, ...) and text. */
mcinv_status mcinv_error_detail(const mcinv_ctx *ctx, int64_t *index, const char **msg);

void mcinv_destroy(mcinv_ctx *ctx);

/* Instrumentation. With timing enabled, every sweep-kernel (K1) and
 * contraction-kernel (K3) launch is bracketed by CUDA events on the launch
 * stream. mcinv_stats returns, since the previous mcinv_stats call: the
 * number of kernels this library launched, and the summed device time (ms)
 * and launch count of K1 and K3 (synchronizes on pending events). */
mcinv_status mcinv_set_timing(mcinv_ctx *ctx, int enable);
mcinv_status mcinv_stats(mcinv_ctx *ctx, int64_t *launches, double *sweep_ms, int64_t *sweep_launches,
                         double *contract_ms, int64_t *contract_launches);

/* Which sweep kernel the last mcinv_run used: 6 = dataflow kernel with
 * TMA-staged plan blocks and the two chains of a Box-Muller pair per thread
 * (sweep6.cu; the default for real C with n <= 200k and no trace), 5 = the
 * dataflow kernel with one chain per thread (sweep5.cu; complex C, trace runs,
 * one chain per CTA), 4 = the same reading its plan through L1, 3 =
 * level-scheduled kernel (C > 32 chains per CTA, deferred pattern pairs, more
 * than 200k rows), 1 = row-by-row kernel (sweep.cu, one thread per chain; the
 * simple reference kernel). chains_per_warp = C, the chains of one CTA;
 * steps_per_sweep = levels D of the row DAG. MCINV_KERNEL=v1|v3|v4|v5|v6 in the
 * environment forces one (MCINV_E_INVALID if it does not apply). */
mcinv_status mcinv_kernel_info(const mcinv_ctx *ctx, int *version, int *chains_per_warp, int64_t *steps_per_sweep);
/* Launch layout of the last run's sweep kernel (the level and dataflow kernels):
 * threads per CTA, chains per thread K (1 or 2; 2 for v6) and CTAs; 0 threads/blocks for
 * the row-by-row kernel. For tests and the bench line. */
mcinv_status mcinv_launch_config(const mcinv_ctx *ctx, int *threads, int *chains_per_thread, int *blocks);

/* ------------------------------------------------------------ test-only */

/* Philox4x32-10 words on the device for `count` counters ctr4[4*count]
 * (host), key = seed; out4[4*count] host. */
mcinv_status mcinv_debug_philox(int device, uint64_t seed, int64_t count, const uint32_t *ctr4,
                                uint32_t *out4);
/* The sweep kernels' Gaussian noise phi(row = ctr4[4t], sweep = ctr4[4t+1], chain =
 * ctr4[4t+2]) for each t (ctr4[4t+3] ignored): output chain%2 of the Box-Muller pair
 * of Philox({row, sweep, chain/2, 0}, seed) (reading R4). Host arrays. */
mcinv_status mcinv_debug_gaussian(int device, uint64_t seed, int64_t count, const uint32_t *ctr4,
                                  double *out);
/* Host-only (no GPU needed): mcinv_create's preprocessing and the level
 * planner of the v3 sweep kernel for C, with the
 * default pattern and an optional Q, for the accumulation of `outputs`.
 * level[n] (may be NULL) receives lev(i); info[7] = {levels D, max items of a
 * phase, fused pattern pairs, deferred pattern pairs, trace items, union
 * entries, slots}. With slots != NULL also the v4 slot schedule for warp
 * groups of slot_R rows and slack slot_L groups:
 * slots[t] = row at slot t or -1 (padding), info[6] = number of slots (E_BUFFER
 * if above slots_capacity). For CPU tests of the planner. */
mcinv_status mcinv_debug_levels(mcinv_dtype dtype, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                const void *values, const int64_t *q_row_ptr, const int32_t *q_col_idx,
                                const void *q_values, unsigned outputs, int32_t *level, int64_t *info,
                                int slot_R, int slot_L, int32_t *slots, int64_t slots_capacity);
/* Host-only (no GPU needed): the dataflow kernels' warp-group schedule as staged in
 * their TMA plan blocks, for R rows per group, W warps per CTA, entries padded to
 * pad_ku (0: default), block entry cap ecap (0: default), with the v6 wait masks
 * (wmask != 0) -- DESIGN.md §3. slot_x[t] = the row at slot t, -1 for padding, -2 - i
 * for the trace item of row i (TRACE in outputs); masks[t] = bit e set when the row
 * waits on its lower-neighbour entry e (< 32). *nslots receives the slot count
 * (E_BUFFER if above capacity). For CPU tests of the schedule and the masks. */
mcinv_status mcinv_debug_blocks(mcinv_dtype dtype, int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                                const void *values, const int64_t *q_row_ptr, const int32_t *q_col_idx,
                                const void *q_values, unsigned outputs, int R, int W, int pad_ku, int ecap, int wmask,
                                int32_t *slot_x, uint32_t *masks, int64_t capacity, int64_t *nslots);
/* Copy the state of chains [chain_begin, chain_begin+chains) (relative to the
 * last run's chain_begin) to host arrays z, w of shape [chains][n] (x2 doubles
 * for C128). Only those chains are copied (one strided copy). Synchronizes. */
mcinv_status mcinv_debug_get_state(mcinv_ctx *ctx, int64_t chain_begin, int64_t chains, void *z, void *w);
/* Per-group accumulator sums of one output of the last run (Eq. 1/C / Eq. tr
 * numerators before the moments): groups [group_begin, group_begin + groups)
 * of this run (0 = the group of its first chain), each count*e doubles, to the
 * host array out[groups][count*e]. Synchronizes. */
mcinv_status mcinv_debug_group_sums(mcinv_ctx *ctx, unsigned output, int64_t group_begin, int64_t groups,
                                    double *out);
/* Overwrite that state from host arrays (same layout); a following run with
 * resume = 1 continues from it. The run's workspace must still be valid. */
mcinv_status mcinv_debug_set_state(mcinv_ctx *ctx, int64_t chain_begin, int64_t chains, const void *z,
                                   const void *w);

#ifdef __cplusplus
}
#endif
#endif /* MCINV_H */
