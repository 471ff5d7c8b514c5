/*
 * oracle.h -- reference (oracle) implementation of the correlated-chains (CC)
 * Monte Carlo inverter of Garcia-Cortes & Cabrillo, arXiv cs/0412107.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this code.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_cs_0412107_b200/), and neither includes the other.
 *
 * Plain, slow, single-threaded C99 in fp64. Every function cites the passage
 * of /root/reference/PAPER.md ("P:<line>") it follows; readings of ambiguous
 * passages are listed in DESIGN.md ("Readings").
 */
#ifndef MCINV_ORACLE_H
#define MCINV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_E_INVALID = 1, ORC_E_ZERO_DIAG = 2, ORC_E_DIAG_DOMAIN = 3,
       ORC_E_DIVERGED = 4, ORC_E_NOMEM = 5 };
enum { ORC_DIAG = 1u, ORC_PATTERN = 2u, ORC_FULL = 4u, ORC_TRACE = 8u };
enum { ORC_NOISE_GAUSS = 0, ORC_NOISE_ZERO = 1, ORC_NOISE_ONE = 2, ORC_NOISE_Z2 = 3 };

typedef struct orc_matrix orc_matrix;

/* Philox4x32-10 block cipher (Salmon et al., SC'11): out = Philox(ctr, key). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Box-Muller transform of one Philox output block (reading R4). */
double orc_gaussian_from_words(const uint32_t r[4]);

/* Both Box-Muller outputs of one block: g[0] the cosine, g[1] the sine branch. */
void orc_gaussian_pair_from_words(const uint32_t r[4], double g[2]);

/* phi(c,k,i) = Box-Muller pair of Philox(ctr={row, sweep, chain/2, 0}, key=seed),
 * the cosine output for even chains, the sine output for odd ones (reading R4). */
double orc_gaussian(uint64_t seed, uint32_t row, uint32_t sweep, uint32_t chain);

/* Z2 noise phi = +-1 (reading R21): the top bit of
 * word 0 of Philox(ctr={row, sweep, chain, 1}, key=seed); 1 -> -1, 0 -> +1. */
double orc_z2(uint64_t seed, uint32_t row, uint32_t sweep, uint32_t chain);

/* Build the split C = L + D + U.  values: n_nz doubles (real) or
 * 2*n_nz doubles (complex, interleaved re,im). Duplicates are summed.
 * Returns ORC_E_ZERO_DIAG (bad_row set) on a zero/missing diagonal and
 * ORC_E_DIAG_DOMAIN on c_ii <= 0 for real C. */
int orc_matrix_build(int64_t n, const int64_t *row_ptr, const int32_t *col,
                     const double *values, int is_complex, orc_matrix **out,
                     int64_t *bad_row);
void orc_matrix_free(orc_matrix *m);
/* Weighting matrix Q of Eq. (tr); same number type as C. */
int orc_set_q(orc_matrix *m, const int64_t *row_ptr, const int32_t *col, const double *values);
/* Selected elements (i,j) of C^-1 to estimate (Eq. 1/C). */
int orc_set_pattern(orc_matrix *m, int64_t count, const int32_t *rows, const int32_t *cols);

typedef struct {
    uint64_t seed;
    int64_t chain_begin, chains;   /* global chain indices [chain_begin, chain_begin+chains) */
    int64_t burn_in, cycles;       /* N and M-N of Eq. (1/C) */
    int64_t sweep_begin;           /* absolute index of the first sweep (noise key) */
    unsigned outputs;              /* ORC_DIAG | ORC_PATTERN | ORC_FULL | ORC_TRACE */
    int noise;                     /* ORC_NOISE_* */
    int use_init;                  /* 0: z = w = 0 (Alg. 1 step 1); 1: z_init / w_init */
} orc_args;

/* Run the CC sampler chain by chain (Eq. 4, 5; Alg. 1 with fixed burn-in).
 * Per-chain sums over the sampling sweeps (not divided) are written to:
 *   diag  [chains][n]       (x2 doubles if complex)  sum_k z_i conj(w_i)
 *   pat   [chains][count]                            sum_k z_i conj(w_j)
 *   full  [chains][n][n]                             sum_k z conj(w)^T
 *   trace [chains]                                   sum_k w^dagger Q z
 *   trace_series [cycles]   the realized w^dagger Q z of each sampling sweep,
 *                           summed over the run's chains (Geyer's series)
 * Any of them may be NULL when not requested. z_out/w_out [chains][n]
 * receive the final state. snap_sweeps (n_snap local sweep indices s, the
 * state after sweep s completes) fill z_snap/w_snap [n_snap][chains][n].
 * On divergence returns ORC_E_DIVERGED with *fail (chain, sweep) set. */
int orc_run(const orc_matrix *m, const orc_args *a,
            const double *z_init, const double *w_init,
            double *diag, double *pat, double *full, double *trace, double *trace_series,
            double *z_out, double *w_out,
            int64_t n_snap, const int64_t *snap_sweeps, double *z_snap, double *w_snap,
            int64_t fail[2]);

/* Geyer's initial positive sequence estimator of a series:
 * out = {mean, gamma_0, sigma2 = m Var(mean), effective length m gamma_0 / sigma2}. */
void orc_geyer(const double *x, int64_t m, double out[4]);

#ifdef __cplusplus
}
#endif
#endif
