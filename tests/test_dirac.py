"""NEXT-3: the free Wilson-Dirac workload of the paper (PAPER.md:784-844,
Tables 3-5) and its exact traces. CPU tests: the generator and the closed
form are pinned against the Clifford algebra, dense inversion and the values
the paper prints; the oracle's CC estimate of tr(L^-1) (Q = I, the paper's
Dirac experiments) agrees with the closed form."""
import os

import numpy as np
import pytest

import workloads as W
from tests import _stats

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "dirac_traces.txt")


def test_gammas_clifford():
    """gamma^mu gamma^nu + gamma^nu gamma^mu = 2 delta_{mu nu}, hermitian
    (the printed gamma^4 and sigma^2 violate it: finding F5, reading R22)."""
    g = W.dirac_gammas()
    for a in range(4):
        assert np.allclose(g[a], g[a].conj().T)
        for b in range(4):
            assert np.allclose(g[a] @ g[b] + g[b] @ g[a], 2.0 * (a == b) * np.eye(4))


def test_structure_fourteen_per_row():
    """rank 4 N^4 and fourteen non-zero elements per row."""
    c = W.dirac(3)
    assert c.n == 4 * 3 ** 4
    assert np.all(np.diff(c.row_ptr) == 14)
    assert np.iscomplexobj(c.val)
    d = c.to_dense()
    assert not np.allclose(d, d.conj().T)  # non-hermitian


@pytest.mark.parametrize("N", [2, 3])
def test_closed_form_equals_dense_inverse(N):
    """The momentum-space closed form of tr(L^-1) is the trace of the dense
    inverse of the generated matrix (pins generator and closed form together)."""
    c = W.dirac(N)
    exact = np.trace(np.linalg.inv(c.to_dense()))
    assert abs(exact.imag) < 1e-9
    assert exact.real == pytest.approx(W.dirac_trace_closed(N), rel=1e-12)


def test_closed_form_matches_paper_tables():
    """Tables 4/5 print the exact traces 413007.84 (N = 18) and 629489.14
    (N = 20) (tests/golden/dirac_traces.txt): the closed form of
    our generator reproduces them to the paper's last digit (within 0.02)."""
    rows = [l.split() for l in open(GOLDEN) if l.strip() and not l.startswith("#")]
    assert len(rows) == 2
    for N, tr in rows:
        assert abs(W.dirac_trace_closed(int(N)) - float(tr)) < 0.02


def test_oracle_cc_trace_of_dirac(orc):
    """The CC estimator of tr(Q L^-1) with Q = I (w^dagger z summed, reading R2;
    Alg. 1 step 8) converges to the closed form on the 2^4 lattice: the
    sampler's spectral condition holds for the Wilson operator at K = 0.1."""
    c = W.dirac(2)
    q = W.identity_q(c.n)
    r = orc.Matrix(c, q=q).run(seed=31, chains=64, burn_in=30, cycles=300, outputs=("trace", "diag"))
    est, se = orc.estimate(r["trace"], 300, group_size=4)
    exact = W.dirac_trace_closed(2)
    _stats.check(np.array([est.real]), np.array([exact]), np.array([se.real]), G=16, what="dirac trace")
    d, sd = orc.estimate(r["diag"], 300, group_size=4)
    assert abs(d.sum() - est) < 1e-9 * abs(est)  # Q = I: trace == sum of the diagonal
