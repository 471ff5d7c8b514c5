/*
 * oracle.c -- plain single-threaded C99 oracle of the correlated-chains (CC)
 * inverter, arXiv cs/0412107 (Garcia-Cortes & Cabrillo).
 *
 * TEST INFRASTRUCTURE ONLY: see oracle.h. Shares no code with the CUDA path.
 * Compile with -ffp-contract=off: the only fused multiply-adds are the
 * explicit fma() calls that define the summation (reading R10).
 *
 * Parity pins: every function below is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_pins.py (Philox KAT + an independent implementation,
 * Gauss-Seidel reduction at zero noise, diagonal/hermitian special cases,
 * dense-LU statistics, exact finite-k expectation, 1/sqrt(samples) slope).
 */
#include "oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ noise ----- */

/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 * easy as 1, 2, 3", SC'11): ten rounds of
 *   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 *   c = (hi1^c1^k0, lo1, hi0^c3^k1, lo0),
 * with the key bumped by the Weyl constants between rounds. The paper only
 * asks for independent noise with E(Phi)=0, E(Phi Phi^dagger)=I
 * (Eq. 5a/5b); the generator is the north_star's choice. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    int r;
    for (r = 0; r < 10; ++r) {
        uint64_t p0, p1;
        uint32_t n0, n1, n2, n3;
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        n1 = (uint32_t)p1;
        n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Box-Muller, cosine branch (reading R4):
 *   u1 = ((r0:r1 >> 11) + 1) 2^-53 in (0,1],  u2 = (r2:r3 >> 11) 2^-53 in [0,1),
 *   phi = sqrt(-2 ln u1) cos(2 pi u2). */
double orc_gaussian_from_words(const uint32_t r[4])
{
    uint64_t a = ((uint64_t)r[0] << 32) | (uint64_t)r[1];
    uint64_t b = ((uint64_t)r[2] << 32) | (uint64_t)r[3];
    double u1 = (double)((a >> 11) + 1u) * 0x1p-53;
    double u2 = (double)(b >> 11) * 0x1p-53;
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* Both outputs of the Box-Muller transform of one block (Box & Muller 1958:
 * two independent N(0,1) from one pair of uniforms; reading R4):
 *   g[0] = sqrt(-2 ln u1) cos(2 pi u2),  g[1] = sqrt(-2 ln u1) sin(2 pi u2). */
void orc_gaussian_pair_from_words(const uint32_t r[4], double g[2])
{
    uint64_t a = ((uint64_t)r[0] << 32) | (uint64_t)r[1];
    uint64_t b = ((uint64_t)r[2] << 32) | (uint64_t)r[3];
    double u1 = (double)((a >> 11) + 1u) * 0x1p-53;
    double u2 = (double)(b >> 11) * 0x1p-53;
    double rad = sqrt(-2.0 * log(u1));
    g[0] = rad * cos(6.283185307179586 * u2);
    g[1] = rad * sin(6.283185307179586 * u2);
}

/* One real N(0,1) per (chain, sweep, row), shared by z_i and w_i: "the noise
 * term in (4) and in (5) are both the same". Chains 2m and 2m+1
 * take the two outputs of one Box-Muller pair, from the Philox block of
 * counter {row, sweep, m, 0} (reading R4): independent N(0,1), as Eq. (5a/5b)
 * require across chains. */
double orc_gaussian(uint64_t seed, uint32_t row, uint32_t sweep, uint32_t chain)
{
    uint32_t ctr[4], key[2], r[4];
    double g[2];
    ctr[0] = row; ctr[1] = sweep; ctr[2] = chain >> 1; ctr[3] = 0u;
    key[0] = (uint32_t)seed; key[1] = (uint32_t)(seed >> 32);
    orc_philox4x32_10(ctr, key, r);
    orc_gaussian_pair_from_words(r, g);
    return g[chain & 1u];
}

/* Z2 noise, the paper's preferred bounded noise "phi = 2B - 1" with B a
 * Bernoulli(1/2) variable: E(phi) = 0, E(phi^2) = 1 as
 * Eq. (5a/5b) require. B is the top bit of word 0 of the Philox block of
 * counter {row, sweep, chain, 1} (4th word 1: a stream disjoint from the
 * Gaussian one; reading R21). */
double orc_z2(uint64_t seed, uint32_t row, uint32_t sweep, uint32_t chain)
{
    uint32_t ctr[4], key[2], r[4];
    ctr[0] = row; ctr[1] = sweep; ctr[2] = chain; ctr[3] = 1u;
    key[0] = (uint32_t)seed; key[1] = (uint32_t)(seed >> 32);
    orc_philox4x32_10(ctr, key, r);
    return (r[0] >> 31) ? -1.0 : 1.0;
}

/* ----------------------------------------------------------- matrix ----- */

typedef struct { double re, im; } cx;

typedef struct {            /* one off-diagonal term of a row list */
    int32_t j;
    cx v;
} term;

struct orc_matrix {
    int64_t n;
    int cplx;
    /* R_i: row i of C without the diagonal, ascending j, values c_ij (Eq. 4)  */
    int64_t *r_ptr; term *r;
    /* K_i: column i of C without the diagonal, ascending j, conj(c_ji) (Eq. 5) */
    int64_t *k_ptr; term *k;
    cx *diag;                /* c_ii */
    cx *delta;               /* 1/c_ii */
    cx *sigma;               /* 1/sqrt(c_ii), principal branch */
    /* Q (Eq. tr), full CSR */
    int64_t *q_ptr; term *q;
    /* pattern */
    int64_t pcount; int32_t *prow, *pcol;
};

static int cmp_term(const void *a, const void *b)
{
    const term *x = (const term *)a, *y = (const term *)b;
    return (x->j > y->j) - (x->j < y->j);
}

/* Sort a row by column and sum duplicates in place; returns new length. */
static int64_t canon_row(term *t, int64_t len)
{
    int64_t i, o = 0;
    qsort(t, (size_t)len, sizeof(term), cmp_term);
    for (i = 0; i < len; ++i) {
        if (o > 0 && t[o - 1].j == t[i].j) {
            t[o - 1].v.re += t[i].v.re;
            t[o - 1].v.im += t[i].v.im;
        } else {
            t[o++] = t[i];
        }
    }
    return o;
}

static int read_csr(int64_t n, const int64_t *rp, const int32_t *col, const double *val,
                    int cplx, int64_t **out_ptr, term **out_t)
{
    int64_t i, e, nnz, o = 0;
    int64_t *ptr;
    term *t;
    if (n < 1 || rp[0] != 0) return ORC_E_INVALID;
    for (i = 0; i < n; ++i)
        if (rp[i + 1] < rp[i]) return ORC_E_INVALID;
    nnz = rp[n];
    ptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    t = (term *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(term));
    if (!ptr || !t) { free(ptr); free(t); return ORC_E_NOMEM; }
    ptr[0] = 0;
    for (i = 0; i < n; ++i) {
        int64_t start = o;
        for (e = rp[i]; e < rp[i + 1]; ++e) {
            if (col[e] < 0 || col[e] >= n) { free(ptr); free(t); return ORC_E_INVALID; }
            t[o].j = col[e];
            t[o].v.re = cplx ? val[2 * e] : val[e];
            t[o].v.im = cplx ? val[2 * e + 1] : 0.0;
            if (!isfinite(t[o].v.re) || !isfinite(t[o].v.im)) { free(ptr); free(t); return ORC_E_INVALID; }
            ++o;
        }
        o = start + canon_row(t + start, o - start);
        ptr[i + 1] = o;
    }
    *out_ptr = ptr;
    *out_t = t;
    return ORC_OK;
}

void orc_matrix_free(orc_matrix *m)
{
    if (!m) return;
    free(m->r_ptr); free(m->r); free(m->k_ptr); free(m->k);
    free(m->diag); free(m->delta); free(m->sigma);
    free(m->q_ptr); free(m->q); free(m->prow); free(m->pcol);
    free(m);
}

/* C = L + D + U: split the diagonal D from the off-diagonal rows
 * R_i (for Eq. 4) and the conjugated columns K_i (for Eq. 5). */
int orc_matrix_build(int64_t n, const int64_t *row_ptr, const int32_t *col,
                     const double *values, int is_complex, orc_matrix **out, int64_t *bad_row)
{
    int64_t *ptr = NULL, i, e, o;
    term *t = NULL;
    int64_t *cnt;
    orc_matrix *m;
    int st = read_csr(n, row_ptr, col, values, is_complex, &ptr, &t);
    if (st) return st;
    m = (orc_matrix *)calloc(1, sizeof(orc_matrix));
    m->n = n;
    m->cplx = is_complex;
    m->diag = (cx *)calloc((size_t)n, sizeof(cx));
    m->delta = (cx *)calloc((size_t)n, sizeof(cx));
    m->sigma = (cx *)calloc((size_t)n, sizeof(cx));
    m->r_ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    m->k_ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    m->r = (term *)malloc((size_t)(ptr[n] + 1) * sizeof(term));
    m->k = (term *)malloc((size_t)(ptr[n] + 1) * sizeof(term));
    cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    /* rows without the diagonal */
    o = 0;
    for (i = 0; i < n; ++i) {
        int have = 0;
        for (e = ptr[i]; e < ptr[i + 1]; ++e) {
            if (t[e].j == i) { m->diag[i] = t[e].v; have = 1; }
            else { m->r[o++] = t[e]; cnt[t[e].j + 1]++; }
        }
        m->r_ptr[i + 1] = o;
        if (!have || (m->diag[i].re == 0.0 && m->diag[i].im == 0.0)) {
            if (bad_row) *bad_row = i;
            free(cnt); free(ptr); free(t); orc_matrix_free(m);
            return ORC_E_ZERO_DIAG;
        }
        if (!is_complex && !(m->diag[i].re > 0.0)) {
            if (bad_row) *bad_row = i;
            free(cnt); free(ptr); free(t); orc_matrix_free(m);
            return ORC_E_DIAG_DOMAIN;
        }
    }
    /* columns: K_i = { (j, conj(c_ji)) : j != i }, ascending j (rows are
     * visited in ascending order, so each column list comes out sorted) */
    for (i = 0; i < n; ++i) m->k_ptr[i + 1] = m->k_ptr[i] + cnt[i + 1];
    for (i = 0; i < n; ++i) cnt[i] = m->k_ptr[i];
    for (i = 0; i < n; ++i) {
        for (e = m->r_ptr[i]; e < m->r_ptr[i + 1]; ++e) {
            int32_t c = m->r[e].j;
            term tt;
            tt.j = (int32_t)i;
            tt.v.re = m->r[e].v.re;
            tt.v.im = -m->r[e].v.im;
            m->k[cnt[c]++] = tt;
        }
    }
    /* delta_i = 1/c_ii and sigma_i = 1/sqrt(c_ii) (Eq. 4); Eq. 5 uses
     * conj(delta_i) and conj(sigma_i) (finding F1; reading R1). */
    for (i = 0; i < n; ++i) {
        if (is_complex) {
            double complex c = m->diag[i].re + I * m->diag[i].im;
            double complex d = 1.0 / c;
            double complex s = 1.0 / csqrt(c);
            m->delta[i].re = creal(d); m->delta[i].im = cimag(d);
            m->sigma[i].re = creal(s); m->sigma[i].im = cimag(s);
        } else {
            m->delta[i].re = 1.0 / m->diag[i].re;
            m->sigma[i].re = 1.0 / sqrt(m->diag[i].re);
        }
    }
    free(cnt); free(ptr); free(t);
    *out = m;
    return ORC_OK;
}

int orc_set_q(orc_matrix *m, const int64_t *row_ptr, const int32_t *col, const double *values)
{
    free(m->q_ptr); free(m->q);
    m->q_ptr = NULL; m->q = NULL;
    return read_csr(m->n, row_ptr, col, values, m->cplx, &m->q_ptr, &m->q);
}

int orc_set_pattern(orc_matrix *m, int64_t count, const int32_t *rows, const int32_t *cols)
{
    int64_t p;
    for (p = 0; p < count; ++p)
        if (rows[p] < 0 || rows[p] >= m->n || cols[p] < 0 || cols[p] >= m->n) return ORC_E_INVALID;
    free(m->prow); free(m->pcol);
    m->pcount = count;
    m->prow = (int32_t *)malloc((size_t)(count > 0 ? count : 1) * sizeof(int32_t));
    m->pcol = (int32_t *)malloc((size_t)(count > 0 ? count : 1) * sizeof(int32_t));
    memcpy(m->prow, rows, (size_t)count * sizeof(int32_t));
    memcpy(m->pcol, cols, (size_t)count * sizeof(int32_t));
    return ORC_OK;
}

/* ------------------------------------------------------------ sweep ----- */

/* Complex fused multiply-add, componentwise (reading R10):
 *   re = fma(a.re, b.re, fma(-a.im, b.im, c.re)),
 *   im = fma(a.re, b.im, fma( a.im, b.re, c.im)). */
static cx cfma(cx a, cx b, cx c)
{
    cx r;
    r.re = fma(a.re, b.re, fma(-a.im, b.im, c.re));
    r.im = fma(a.re, b.im, fma(a.im, b.re, c.im));
    return r;
}

static double noise(const orc_args *a, int64_t i, int64_t k, int64_t c)
{
    if (a->noise == ORC_NOISE_ZERO) return 0.0;
    if (a->noise == ORC_NOISE_ONE) return 1.0;
    if (a->noise == ORC_NOISE_Z2) return orc_z2(a->seed, (uint32_t)i, (uint32_t)k, (uint32_t)c);
    return orc_gaussian(a->seed, (uint32_t)i, (uint32_t)k, (uint32_t)c);
}

/* One sweep k of Eq. (4) and Eq. (5), rows i = 0..n-1 ascending,
 * z and w updated in place so j < i reads cycle-k values and j > i reads
 * cycle k-1 values ("updates simultaneously each element"):
 *   z_i = sigma_i phi - delta_i sum_{j!=i} c_ij z_j
 *   w_i = conj(sigma_i) phi - conj(delta_i) sum_{j!=i} conj(c_ji) w_j
 * with the sums accumulated by serial fma from 0 in ascending j. */
static void sweep(const orc_matrix *m, cx *z, cx *w, const orc_args *a, int64_t k, int64_t c)
{
    int64_t i, e;
    for (i = 0; i < m->n; ++i) {
        double phi = noise(a, i, k, c);
        cx az = {0.0, 0.0}, aw = {0.0, 0.0};
        cx nd, ndc, sp, spc;
        if (m->cplx) {
            for (e = m->r_ptr[i]; e < m->r_ptr[i + 1]; ++e) az = cfma(m->r[e].v, z[m->r[e].j], az);
            for (e = m->k_ptr[i]; e < m->k_ptr[i + 1]; ++e) aw = cfma(m->k[e].v, w[m->k[e].j], aw);
            nd.re = -m->delta[i].re; nd.im = -m->delta[i].im;      /* -delta_i */
            ndc.re = -m->delta[i].re; ndc.im = m->delta[i].im;     /* -conj(delta_i) */
            sp.re = m->sigma[i].re * phi; sp.im = m->sigma[i].im * phi;
            spc.re = m->sigma[i].re * phi; spc.im = -(m->sigma[i].im * phi);
            z[i] = cfma(nd, az, sp);
            w[i] = cfma(ndc, aw, spc);
        } else {
            for (e = m->r_ptr[i]; e < m->r_ptr[i + 1]; ++e) az.re = fma(m->r[e].v.re, z[m->r[e].j].re, az.re);
            for (e = m->k_ptr[i]; e < m->k_ptr[i + 1]; ++e) aw.re = fma(m->k[e].v.re, w[m->k[e].j].re, aw.re);
            z[i].re = fma(-m->delta[i].re, az.re, m->sigma[i].re * phi);
            w[i].re = fma(-m->delta[i].re, aw.re, m->sigma[i].re * phi);
            z[i].im = 0.0;
            w[i].im = 0.0;
        }
    }
}

/* z_i conj(w_j), the summand of Eq. (1/C). */
static cx zwc(cx z, cx w)
{
    cx r;
    r.re = z.re * w.re + z.im * w.im;
    r.im = z.im * w.re - z.re * w.im;
    return r;
}

static int diverged(const cx *z, const cx *w, int64_t n)
{
    int64_t i;
    for (i = 0; i < n; ++i) {
        double v[4] = {z[i].re, z[i].im, w[i].re, w[i].im};
        int q;
        for (q = 0; q < 4; ++q)
            if (!isfinite(v[q]) || fabs(v[q]) > 1e12) return 1;
    }
    return 0;
}

static void put(double *dst, int64_t idx, cx v, int cplx)
{
    if (cplx) { dst[2 * idx] += v.re; dst[2 * idx + 1] += v.im; }
    else dst[idx] += v.re;
}

/* Algorithm 1 with a fixed burn-in N: for each chain, start at
 * z = w = 0 (step 1), run N + (M-N) sweeps (steps 3 and 7), and after every
 * sampling sweep accumulate the estimators (step 8). Accumulation happens
 * after the sweep completes, from the stored vectors. The trace uses
 * w^dagger Q z, whose expectation is tr(Q C^-1) (finding F2; DESIGN.md
 * reading R2), instead of the printed z^dagger Q w. */
int orc_run(const orc_matrix *m, const orc_args *a,
            const double *z_init, const double *w_init,
            double *diag, double *pat, double *full, double *trace, double *trace_series,
            double *z_out, double *w_out,
            int64_t n_snap, const int64_t *snap_sweeps, double *z_snap, double *w_snap,
            int64_t fail[2])
{
    const int64_t n = m->n, e = m->cplx ? 2 : 1;
    int64_t ci, s, i, j, p, q;
    const int64_t total = a->burn_in + a->cycles;
    cx *z = (cx *)malloc((size_t)n * sizeof(cx));
    cx *w = (cx *)malloc((size_t)n * sizeof(cx));
    if (!z || !w) { free(z); free(w); return ORC_E_NOMEM; }
    if ((a->outputs & ORC_TRACE) && !m->q_ptr) { free(z); free(w); return ORC_E_INVALID; }
    if ((a->outputs & ORC_PATTERN) && !m->prow) { free(z); free(w); return ORC_E_INVALID; }
    for (ci = 0; ci < a->chains; ++ci) {
        const int64_t c = a->chain_begin + ci;
        for (i = 0; i < n; ++i) {
            if (a->use_init) {
                z[i].re = z_init[(ci * n + i) * e]; z[i].im = m->cplx ? z_init[(ci * n + i) * e + 1] : 0.0;
                w[i].re = w_init[(ci * n + i) * e]; w[i].im = m->cplx ? w_init[(ci * n + i) * e + 1] : 0.0;
            } else {
                z[i].re = z[i].im = w[i].re = w[i].im = 0.0;
            }
        }
        for (s = 0; s < total; ++s) {
            sweep(m, z, w, a, a->sweep_begin + s, c);
            if (diverged(z, w, n)) {
                if (fail) { fail[0] = c; fail[1] = a->sweep_begin + s; }
                free(z); free(w);
                return ORC_E_DIVERGED;
            }
            for (q = 0; q < n_snap; ++q) {
                if (snap_sweeps[q] != s) continue;
                for (i = 0; i < n; ++i) {
                    int64_t o = ((q * a->chains + ci) * n + i) * e;
                    z_snap[o] = z[i].re; w_snap[o] = w[i].re;
                    if (m->cplx) { z_snap[o + 1] = z[i].im; w_snap[o + 1] = w[i].im; }
                }
            }
            if (s < a->burn_in) continue;
            if ((a->outputs & ORC_DIAG) && diag)
                for (i = 0; i < n; ++i) put(diag, ci * n + i, zwc(z[i], w[i]), m->cplx);
            if ((a->outputs & ORC_PATTERN) && pat)
                for (p = 0; p < m->pcount; ++p)
                    put(pat, ci * m->pcount + p, zwc(z[m->prow[p]], w[m->pcol[p]]), m->cplx);
            if ((a->outputs & ORC_FULL) && full)
                for (i = 0; i < n; ++i)
                    for (j = 0; j < n; ++j)
                        put(full, (ci * n + i) * n + j, zwc(z[i], w[j]), m->cplx);
            if ((a->outputs & ORC_TRACE) && trace) {
                /* w^dagger Q z = sum_i conj(w_i) sum_j Q_ij z_j */
                cx t = {0.0, 0.0};
                for (i = 0; i < n; ++i) {
                    cx qz = {0.0, 0.0}, wc;
                    for (p = m->q_ptr[i]; p < m->q_ptr[i + 1]; ++p) {
                        cx qq = m->q[p].v, zz = z[m->q[p].j];
                        qz.re += qq.re * zz.re - qq.im * zz.im;
                        qz.im += qq.re * zz.im + qq.im * zz.re;
                    }
                    wc = zwc(qz, w[i]);   /* qz * conj(w_i) */
                    t.re += wc.re; t.im += wc.im;
                }
                put(trace, ci, t, m->cplx);
                /* the realized value of this sampling sweep, summed over the run's chains */
                if (trace_series) put(trace_series, s - a->burn_in, t, m->cplx);
            }
        }
        if (z_out && w_out) {
            for (i = 0; i < n; ++i) {
                z_out[(ci * n + i) * e] = z[i].re; w_out[(ci * n + i) * e] = w[i].re;
                if (m->cplx) { z_out[(ci * n + i) * e + 1] = z[i].im; w_out[(ci * n + i) * e + 1] = w[i].im; }
            }
        }
    }
    free(z); free(w);
    return ORC_OK;
}

/* ------------------------------------------------------------ Geyer ----- */

/* Effective sample size of a serially correlated series x[0..m-1] by Geyer's
 * initial positive sequence estimator (Geyer 1992, "Practical Markov chain
 * Monte Carlo", the method the paper uses for its standard errors, P:354-360,
 * P:553-557): with the mean xbar and the lag-k autocovariances
 *   gamma_k = (1/m) sum_{t=0}^{m-1-k} (x_t - xbar)(x_{t+k} - xbar),
 * the pair sums Gamma_j = gamma_{2j} + gamma_{2j+1} are summed for
 * j = 0, 1, ... while positive (stopping before the first Gamma_j <= 0 or when
 * 2j + 1 reaches m), the asymptotic variance of the mean times m is
 *   sigma2 = -gamma_0 + 2 sum_j Gamma_j,
 * and ESS = m gamma_0 / sigma2, so that SE(mean) = sqrt(gamma_0 / ESS) =
 * sqrt(sigma2 / m) (the paper's "MC St. error" = sqrt(Var / Eff. length),
 * Table 2). out = {xbar, gamma_0, sigma2, ESS}. */
void orc_geyer(const double *x, int64_t m, double out[4])
{
    int64_t t, k, j;
    double xbar = 0.0, g0, sigma2;
    for (t = 0; t < m; ++t) xbar += x[t];
    xbar /= (double)m;
    g0 = 0.0;
    for (t = 0; t < m; ++t) g0 += (x[t] - xbar) * (x[t] - xbar);
    g0 /= (double)m;
    sigma2 = -g0;
    for (j = 0; 2 * j + 1 < m; ++j) {
        double gam[2];
        for (k = 0; k < 2; ++k) {
            int64_t lag = 2 * j + k;
            double acc = 0.0;
            for (t = 0; t + lag < m; ++t) acc += (x[t] - xbar) * (x[t + lag] - xbar);
            gam[k] = acc / (double)m;
        }
        if (!(gam[0] + gam[1] > 0.0)) break;
        sigma2 += 2.0 * (gam[0] + gam[1]);
    }
    out[0] = xbar;
    out[1] = g0;
    out[2] = sigma2;
    out[3] = sigma2 > 0.0 ? (double)m * g0 / sigma2 : 0.0;
}
