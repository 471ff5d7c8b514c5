"""Seeded synthetic inputs for the correlated-chains (CC) inverter.

This module is the ONLY code shared by the oracle tests (``oracle/``) and the
CUDA path (``paper_cs_0412107_b200``). It builds input matrices C, weighting
matrices Q, and run parameters. It holds none of the method's arithmetic: no
noise, no sweep, no estimator. Everything is numpy (PCG64) seeded, so both
sides receive bit-identical CSR arrays.

Recipes follow SURVEY.md §8(c) rows 16-19 and BASELINE.json ``configs``;
DESIGN.md §"Input recipe" states them in prose. The paper's own datasets
(Wu-Schaeffer pedigrees, Table 1; free Dirac lattices,
PAPER.md:846-878, Table 3) are not in the container; configs 2/4 stand in
for the former and configs 3/5 for the latter.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional

import numpy as np
import scipy.sparse as sp

__all__ = [
    "CSR", "RunSpec", "dense_config1", "pedigree", "lattice", "random_q",
    "random_dense", "diagonal", "config", "CONFIGS", "RUN_SEED_BASE", "dirac", "dirac_gammas",
    "dirac_trace_closed", "identity_q",
]

RUN_SEED_BASE = 0x5EED0000


@dataclasses.dataclass
class CSR:
    """Compressed sparse row matrix; 0-based; columns ascending, no duplicates.

    ``val`` is float64 (dtype "f64") or complex128 (dtype "c128").
    """
    n: int
    row_ptr: np.ndarray  # int64[n+1]
    col: np.ndarray      # int32[nnz]
    val: np.ndarray      # float64[nnz] or complex128[nnz]

    @property
    def dtype(self) -> str:
        return "c128" if np.iscomplexobj(self.val) else "f64"

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    def to_scipy(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.val, self.col, self.row_ptr), shape=(self.n, self.n))

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.row_ptr, self.col, self.val):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    @staticmethod
    def from_scipy(m) -> "CSR":
        m = sp.csr_matrix(m)
        m.sum_duplicates()
        m.sort_indices()
        return CSR(m.shape[0], m.indptr.astype(np.int64), m.indices.astype(np.int32),
                   np.ascontiguousarray(m.data))

    @staticmethod
    def from_dense(a: np.ndarray, keep_zeros_on_diag: bool = True) -> "CSR":
        a = np.asarray(a)
        n = a.shape[0]
        mask = a != 0
        if keep_zeros_on_diag:
            mask |= np.eye(n, dtype=bool)
        rows, cols = np.nonzero(mask)
        rp = np.zeros(n + 1, np.int64)
        np.add.at(rp, rows + 1, 1)
        rp = np.cumsum(rp)
        return CSR(n, rp, cols.astype(np.int32), np.ascontiguousarray(a[rows, cols]))


@dataclasses.dataclass
class RunSpec:
    """Run parameters of one BASELINE.json config."""
    chains: int
    burn_in: int
    cycles: int
    outputs: tuple  # subset of ("diag", "pattern", "full", "trace")
    seed: int
    group_size: int = 32


# ---------------------------------------------------------------- generators

def dense_config1(n: int = 64, seed: int = 1001) -> CSR:
    """Config 1 (BASELINE.json configs[0]).

    c_ii = 1 + U(0,1); off-diagonals iid U(-1,1) rescaled so that the row's
    absolute off-diagonal sum is 0.5 c_ii. Dense, real, non-symmetric.
    """
    rng = np.random.default_rng(seed)
    d = 1.0 + rng.random(n)
    a = rng.uniform(-1.0, 1.0, size=(n, n))
    np.fill_diagonal(a, 0.0)
    s = np.abs(a).sum(axis=1)
    a *= (0.5 * d / s)[:, None]
    np.fill_diagonal(a, d)
    return CSR.from_dense(a)


def pedigree(n: int, seed: int, mate: bool = True, asym: float = 0.3,
             dominance: float = 1.1) -> CSR:
    """Pedigree / mixed-model-like real non-symmetric C (configs 2 and 4).

    SURVEY §8(c) row 16, modelled on Wu-Schaeffer rules:
    rows 0 and 1 are founders; row i >= 2 picks two distinct parents p1, p2
    uniformly in [0, i). Entries (i,p) = -0.5 and (p,i) = -0.5 (1 + U(-asym,
    asym)); with ``mate`` a symmetric sire-dam link (p1,p2) = (p2,p1) = -0.25
    (rule 4) gives the ~7 nnz/row of BASELINE.json (finding F3).
    Duplicates are summed. Then c_ii = dominance * sum_j!=i |c_ij| (strict row
    diagonal dominance, so sp(T), sp(S) < 1).
    """
    rng = np.random.default_rng(seed)
    i = np.arange(2, n, dtype=np.int64)
    p1 = np.floor(rng.random(i.size) * i).astype(np.int64)
    p2 = np.floor(rng.random(i.size) * (i - 1)).astype(np.int64)
    p2 = p2 + (p2 >= p1)
    u1 = rng.uniform(-asym, asym, size=i.size)
    u2 = rng.uniform(-asym, asym, size=i.size)
    rows = [i, p1, i, p2]
    cols = [p1, i, p2, i]
    vals = [np.full(i.size, -0.5), -0.5 * (1.0 + u1), np.full(i.size, -0.5), -0.5 * (1.0 + u2)]
    if mate:
        rows += [p1, p2]
        cols += [p2, p1]
        vals += [np.full(i.size, -0.25), np.full(i.size, -0.25)]
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals)
    off = sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr()
    off.sum_duplicates()
    rowsum = np.asarray(abs(off).sum(axis=1)).ravel()
    diag = dominance * rowsum
    diag[diag == 0.0] = 1.0
    m = off + sp.diags(diag, format="csr")
    return CSR.from_scipy(m)


def lattice(L: int, d: int, kappa: float, seed: int, back: float = 0.6,
            pure_gauge: bool = False, free: bool = False) -> CSR:
    """Complex non-hermitian periodic hopping matrix (configs 3 and 5).

    SURVEY §8(c) row 17, standing in for the Dirac operator of PAPER.md:784-844:
    site x = x0 + L x1 + L^2 x2 + ... (x0 fastest). Each link (x, mu) carries
    a U(1) phase U = e^{i theta}; C[x, x+mu] = -kappa U, C[x+mu, x] =
    -back * kappa * conj(U) (the conjugate of the same link); diagonal 1.
    ``pure_gauge`` uses U_mu(x) = e^{i(g_x - g_{x+mu})} (finding F4), whose
    C^-1 diagonal has the closed form in ``lattice_pure_gauge_diag``.
    ``free`` sets every U = 1.
    """
    rng = np.random.default_rng(seed)
    n = L ** d
    x = np.arange(n, dtype=np.int64)
    coords = [(x // (L ** mu)) % L for mu in range(d)]
    if pure_gauge:
        g = rng.uniform(0.0, 2.0 * np.pi, size=n)
    rows, cols, vals = [x], [x], [np.ones(n, np.complex128)]
    for mu in range(d):
        xf = x + (((coords[mu] + 1) % L) - coords[mu]) * (L ** mu)
        if free:
            u = np.ones(n, np.complex128)
        elif pure_gauge:
            u = np.exp(1j * (g[x] - g[xf]))
        else:
            u = np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, size=n))
        rows += [x, xf]
        cols += [xf, x]
        vals += [-kappa * u, -back * kappa * np.conj(u)]
    m = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    return CSR.from_scipy(m)


def lattice_pure_gauge_diag(L: int, d: int, kappa: float, back: float = 0.6) -> float:
    """Closed form of every diagonal entry of C^-1 for the pure-gauge lattice.

    C = G C0 G^dagger with G unitary diagonal, so diag(C^-1) = diag(C0^-1) =
    (1/n) sum_p 1/lambda(p), lambda(p) = 1 - kappa sum_mu (e^{i p_mu} + back
    e^{-i p_mu}), p_mu = 2 pi k / L (finding F4).
    This is a property of the INPUT (a spectral identity), not of the method.
    """
    ks = np.arange(L) * 2.0 * np.pi / L
    grids = np.meshgrid(*([ks] * d), indexing="ij")
    lam = 1.0 - kappa * sum(np.exp(1j * p) + back * np.exp(-1j * p) for p in grids)
    v = np.mean(1.0 / lam)
    return float(v.real)


# Hermitian Euclidean gamma matrices (Dirac basis): the paper's printed gamma^i =
# [[0, sigma^i], [sigma^i, 0]] with the Pauli matrices, and gamma^4 =
# diag(1, 1, -1, -1) instead of the printed [[0, 1], [1, 0]], which commutes
# with the gamma^i and violates the anticommutator of PAPER.md:731 (finding
# F5; reading R22). This set satisfies it and gives the paper's
# "fourteen non zero elements per row".
_SIGMA = [np.array([[0, 1], [1, 0]], np.complex128), np.array([[0, -1j], [1j, 0]], np.complex128),
          np.array([[1, 0], [0, -1]], np.complex128)]


def dirac_gammas():
    g = []
    for s_ in _SIGMA:
        m = np.zeros((4, 4), np.complex128)
        m[:2, 2:] = s_
        m[2:, :2] = s_
        g.append(m)
    g.append(np.diag([1.0, 1.0, -1.0, -1.0]).astype(np.complex128))
    return g


def dirac(N: int, K: float = 0.1) -> CSR:
    """Free Wilson-Dirac matrix of PAPER.md Eq. (disDirac), P:784-796 (NEXT-3):
    L = 1 + K sum_mu [(1 + gamma^mu) delta_{m+mu, n} + (1 - gamma^mu) delta_{m-mu, n}]
    on a periodic N^4 lattice, with the index map of P:826-833: row = site +
    N^4 * spinor, site = x1 + N (x2 + N (x3 + N x0)) (spinor slowest);
    direction mu = 1, 2, 3, 4 hops along x1, x2, x3, x0 (gamma^1 pairs with
    the first index). Complex, non-hermitian, n = 4 N^4, 14 nnz/row.
    """
    V = N ** 4
    site = np.arange(V, dtype=np.int64)
    coord = [(site // N ** k) % N for k in range(4)]
    gam = dirac_gammas()
    one = np.eye(4)
    rows, cols, vals = [], [], []
    for r in range(4):  # the diagonal
        rows.append(site + V * r)
        cols.append(site + V * r)
        vals.append(np.ones(V, np.complex128))
    for mu in range(4):
        for sgn in (+1, -1):
            nb = site + (((coord[mu] + sgn) % N) - coord[mu]) * N ** mu
            m = K * (one + sgn * gam[mu])
            for r in range(4):
                for rp in range(4):
                    if m[r, rp] != 0:
                        rows.append(site + V * r)
                        cols.append(nb + V * rp)
                        vals.append(np.full(V, m[r, rp], np.complex128))
    n = 4 * V
    mat = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                        shape=(n, n)).tocsr()
    return CSR.from_scipy(mat)


def dirac_trace_closed(N: int, K: float = 0.1) -> float:
    """tr(L^-1) of the free Wilson-Dirac matrix: L(p) = a + i gamma.b with a =
    1 + 2K sum cos p_mu, b_mu = 2K sin p_mu, p_mu = 2 pi k / N, so the spinor
    trace of L(p)^-1 is 4a / (a^2 + |b|^2) (Clifford relations), summed over
    momenta (finding F5). A property of the INPUT, not of the method; the paper
    prints 413007.84 (N = 18) and 629489.14 (N = 20)."""
    p = 2.0 * np.pi * np.arange(N) / N
    P = np.meshgrid(p, p, p, p, indexing="ij")
    a = 1.0 + 2.0 * K * sum(np.cos(x) for x in P)
    b2 = sum((2.0 * K * np.sin(x)) ** 2 for x in P)
    return float(np.sum(4.0 * a / (a * a + b2)))


def identity_q(n: int, complex_: bool = True) -> CSR:
    """Q = I: tr(Q C^-1) = tr(C^-1), the paper's Dirac experiments."""
    v = np.ones(n, np.complex128 if complex_ else np.float64)
    return CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), v)


def random_q(n: int, seed: int = 2005, per_row: int = 4, complex_: bool = True) -> CSR:
    """Seeded random sparse Q (config 5): ``per_row``
    distinct uniform columns per row, entries re, im ~ U(-1, 1)."""
    rng = np.random.default_rng(seed)
    k = min(per_row, n)
    cols = np.argsort(rng.random((n, n)), axis=1)[:, :k] if n <= 512 else \
        _distinct_cols(rng, n, k)
    rows = np.repeat(np.arange(n), k)
    v = rng.uniform(-1, 1, size=n * k)
    if complex_:
        v = v + 1j * rng.uniform(-1, 1, size=n * k)
    m = sp.coo_matrix((v, (rows, cols.ravel())), shape=(n, n)).tocsr()
    return CSR.from_scipy(m)


def _distinct_cols(rng, n, k):
    cols = rng.integers(0, n, size=(n, k))
    for _ in range(64):
        s = np.sort(cols, axis=1)
        dup = np.any(s[:, 1:] == s[:, :-1], axis=1)
        if not dup.any():
            return cols
        cols[dup] = rng.integers(0, n, size=(int(dup.sum()), k))
    raise RuntimeError("could not draw distinct columns")


def random_dense(n: int, seed: int, complex_: bool = False, ratio: float = 0.5,
                 hermitian: bool = False, density: float = 1.0,
                 diag_phase: Optional[float] = None) -> CSR:
    """Small test matrices: diagonally dominant with off-diagonal row sum =
    ``ratio`` * |c_ii|. ``hermitian`` symmetrises (real positive diagonal).
    ``diag_phase`` puts every diagonal at angle diag_phase (e.g. pi puts it
    on the negative real axis, the branch-cut case of finding F1)."""
    rng = np.random.default_rng(seed)
    d = 1.0 + rng.random(n)
    a = rng.uniform(-1, 1, size=(n, n))
    if complex_:
        a = a + 1j * rng.uniform(-1, 1, size=(n, n))
    if density < 1.0:
        a = a * (rng.random((n, n)) < density)
    np.fill_diagonal(a, 0)
    if hermitian:
        a = np.triu(a)
        a = a + a.conj().T
    s = np.abs(a).sum(axis=1)
    s[s == 0] = 1.0
    a = a * (ratio * d / s)[:, None] if not hermitian else a * (ratio * d.min() / s.max())
    if complex_ and diag_phase is not None:
        if diag_phase == np.pi:
            # exactly on the negative real axis with a +0 imaginary part
            dd = (-d).astype(np.complex128)
        else:
            dd = d * np.exp(1j * diag_phase)
        a = a.astype(np.complex128)
        np.fill_diagonal(a, dd)
    else:
        np.fill_diagonal(a, d)
    return CSR.from_dense(a)


def diagonal(d) -> CSR:
    d = np.asarray(d)
    n = d.size
    return CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
               np.ascontiguousarray(d))


# ------------------------------------------------------------------ configs

CONFIGS = {
    1: dict(name="cfg1_dense64_f64", dtype="f64",
            run=RunSpec(chains=64, burn_in=100, cycles=1000, outputs=("full",),
                        seed=RUN_SEED_BASE + 1, group_size=1)),
    2: dict(name="cfg2_pedigree20k_f64", dtype="f64",
            run=RunSpec(chains=1024, burn_in=200, cycles=2000, outputs=("diag", "pattern"),
                        seed=RUN_SEED_BASE + 2, group_size=32)),
    3: dict(name="cfg3_lattice2d_L64_c128", dtype="c128",
            run=RunSpec(chains=2048, burn_in=200, cycles=2000, outputs=("full",),
                        seed=RUN_SEED_BASE + 3, group_size=32)),
    4: dict(name="cfg4_pedigree1M_f64", dtype="f64",
            run=RunSpec(chains=8192, burn_in=100, cycles=500, outputs=("diag",),
                        seed=RUN_SEED_BASE + 4, group_size=32)),
    5: dict(name="cfg5_lattice4d_16_c128", dtype="c128",
            run=RunSpec(chains=16384, burn_in=200, cycles=1000, outputs=("diag", "trace"),
                        seed=RUN_SEED_BASE + 5, group_size=32)),
}


def config(k: int, pure_gauge: bool = False):
    """Return (C, Q or None, RunSpec) for BASELINE.json configs[k-1].

    Matrix seed 1000 + k, Q seed 2005, run seed 0x5EED0000 + k
    (SURVEY §8(d) row d2)."""
    spec = CONFIGS[k]
    run = dataclasses.replace(spec["run"])
    q = None
    if k == 1:
        c = dense_config1(64, 1000 + k)
    elif k == 2:
        c = pedigree(20000, 1000 + k)
    elif k == 3:
        c = lattice(64, 2, 0.2, 1000 + k, pure_gauge=pure_gauge)
    elif k == 4:
        c = pedigree(1_000_000, 1000 + k)
    elif k == 5:
        c = lattice(16, 4, 0.1, 1000 + k, pure_gauge=pure_gauge)
        q = random_q(c.n, 2005, 4, complex_=True)
    else:
        raise KeyError(k)
    return c, q, run
