"""Pins of the oracle (oracle/oracle.c) to things other than itself.

Every test here is CPU-only. Each pin names the passage of PAPER.md ("P:n")
or the mathematical fact it checks, and is chosen so that a plausible mistake
(dropped term, wrong sign or index, transposed operand, wrong noise branch,
off-by-one in burn-in) fails at least one of them:

* Philox words       : published KAT vectors + PyTorch's independent engine
* Box-Muller         : closed-form values at chosen words; KS normality
* sweep structure    : zero noise == textbook Gauss-Seidel (Eq. 12)
* transposition      : hand-unrolled n=3 recurrence
* noise coefficient  : diagonal C closed form incl. the branch cut (F1)
* hermitian collapse : w == z exactly
* coupling identity  : difference of two starts == GS (Eq. 12)
* expectation        : exact finite-k mean P_k (derived from Eq. zk/wk)
* stationary target  : dense LU statistics (Eq. 1/C), 1/sqrt(samples) slope
* trace              : w^dagger Q z -> tr(QC^-1) (Eq. tr, finding F2)
* one-draw GS        : hermitian PD C, independent numpy Eq. (2) sampler
* lattice            : pure-gauge closed form (finding F4)
* bookkeeping        : resume / chain-subset equivalence, duplicates, errors
"""
import os
import shutil
import subprocess

import numpy as np
import pytest
import scipy.linalg as sla

import workloads as W
from tests import _stats

HERE = os.path.dirname(os.path.abspath(__file__))


# ------------------------------------------------------------------ noise

def _kat():
    rows = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(orc):
    kat = _kat()
    assert len(kat) == 3
    for ctr, key, out in kat:
        assert list(orc.philox(ctr, key)) == out


def test_philox_matches_pytorch_engine(orc, tmp_path):
    """Bit-exact against at::philox_engine (an independent implementation)."""
    import torch
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = tmp_path / "philox_ref"
    subprocess.check_call([gxx, "-std=c++17", "-O1", "-I", inc, "-o", str(exe),
                           os.path.join(HERE, "native", "philox_torch_ref.cpp")])
    rng = np.random.default_rng(7)
    cases = rng.integers(0, 2**32, size=(400, 6), dtype=np.uint64).tolist()
    cases += [[i, k, c, 0, 0x5EED0002, 0] for i in (0, 1, 19999) for k in (0, 1, 2199) for c in (0, 1023)]
    inp = "\n".join(" ".join(str(int(x)) for x in cse) for cse in cases) + "\n"
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    for cse, line in zip(cases, out):
        ref = [int(x) for x in line.split()]
        assert list(orc.philox(cse[:4], cse[4:6])) == ref, cse


def test_box_muller_closed_forms(orc):
    """Reading R4: u1 = ((r0:r1 >> 11) + 1) 2^-53, u2 = (r2:r3 >> 11) 2^-53,
    phi = sqrt(-2 ln u1) cos(2 pi u2); checked at words with exact u's."""
    # u1 = 2^-53, u2 = 0 -> sqrt(106 ln 2)
    assert orc.gaussian_from_words([0, 0, 0, 0]) == pytest.approx(np.sqrt(106 * np.log(2)), rel=1e-15)
    # u1 = 1 -> phi = 0 whatever u2
    assert orc.gaussian_from_words([0xFFFFFFFF, 0xFFFFFFFF, 123, 456]) == 0.0
    # u1 = 1/2 (a >> 11 = 2^52 - 1), u2 = 1/2 (b >> 11 = 2^52) -> -sqrt(2 ln 2)
    a = (2**52 - 1) << 11
    b = 2**52 << 11
    w = [a >> 32, a & 0xFFFFFFFF, b >> 32, b & 0xFFFFFFFF]
    assert orc.gaussian_from_words(w) == pytest.approx(-np.sqrt(2 * np.log(2)), rel=1e-15)
    # u2 = 1/8 -> cos(pi/4); the low 11 bits are discarded
    b = (2**50 << 11) | 0x7FF
    w = [a >> 32, a & 0xFFFFFFFF, b >> 32, b & 0xFFFFFFFF]
    assert orc.gaussian_from_words(w) == pytest.approx(np.sqrt(2 * np.log(2)) * np.sqrt(0.5), rel=1e-15)


def test_box_muller_pair_closed_forms(orc):
    """The pair (reading R4): g0 = sqrt(-2 ln u1) cos(2 pi u2) (the cosine output
    above), g1 = sqrt(-2 ln u1) sin(2 pi u2); exact u's again."""
    rad = np.sqrt(2 * np.log(2))
    a = (2**52 - 1) << 11  # u1 = 1/2
    for u2_bits, want_c, want_s in ((2**50, np.sqrt(0.5), np.sqrt(0.5)),   # u2 = 1/8
                                    (2**51, 0.0, 1.0),                    # u2 = 1/4
                                    (3 * 2**51, 0.0, -1.0),               # u2 = 3/4
                                    (2**52, -1.0, 0.0),                   # u2 = 1/2
                                    (0, 1.0, 0.0)):                       # u2 = 0
        b = u2_bits << 11
        w = [a >> 32, a & 0xFFFFFFFF, b >> 32, b & 0xFFFFFFFF]
        g0, g1 = orc.gaussian_pair_from_words(w)
        assert g0 == orc.gaussian_from_words(w)
        assert g0 == pytest.approx(rad * want_c, rel=1e-15, abs=1e-15)
        assert g1 == pytest.approx(rad * want_s, rel=1e-15, abs=1e-15)
    # one radius for both outputs: g0^2 + g1^2 = -2 ln u1 at random words
    rng = np.random.default_rng(3)
    for w in rng.integers(0, 2**32, size=(200, 4), dtype=np.uint64).tolist():
        g0, g1 = orc.gaussian_pair_from_words(w)
        aa = (int(w[0]) << 32 | int(w[1])) >> 11
        u1 = (aa + 1) * 2.0**-53
        assert g0 * g0 + g1 * g1 == pytest.approx(-2 * np.log(u1), rel=1e-13)


def test_gaussian_counter_layout(orc):
    """Reading R4's counter layout, pinned on the CPU: the noise of (chain c,
    sweep k, row i) is output c mod 2 (cosine for even, sine for odd chains)
    of the Box-Muller pair of the Philox block of counter {i, k, c / 2, 0}
    under key {seed lo, seed hi} -- composed here from the separately pinned
    pieces (KAT-pinned Philox, closed-form-pinned Box-Muller pair), so a
    swapped or misplaced counter word, or a wrong branch, inside orc_gaussian
    fails."""
    rng = np.random.default_rng(11)
    for seed in (0, 0x5EED0002, 2**64 - 1, 0x123456789ABCDEF):
        key = [seed & 0xFFFFFFFF, seed >> 32]
        for i, k, c in rng.integers(0, 2**32, size=(40, 3), dtype=np.uint64).tolist() + [[0, 0, 0], [5, 0, 1]]:
            pair = orc.gaussian_pair_from_words(orc.philox([i, k, c >> 1, 0], key))
            assert orc.gaussian(seed, i, k, c) == pair[c & 1]
            assert orc.gaussian(seed, i, k, c ^ 1) == pair[(c & 1) ^ 1]  # the partner chain
            # a transposed layout gives a different value
            if len({i, k, c >> 1}) == 3:
                assert orc.gaussian(seed, i, k, c) != orc.gaussian_pair_from_words(
                    orc.philox([k, i, c >> 1, 0], key))[c & 1]


def test_gaussian_is_standard_normal(orc):
    """E(Phi) = 0, E(Phi Phi^T) = I (Eq. 5a/5b)."""
    from scipy import stats
    seed = 0x5EED0002
    x = np.array([orc.gaussian(seed, i, k, c) for c in range(8) for k in range(25) for i in range(200)])
    assert abs(x.mean()) < 5 / np.sqrt(x.size)
    assert abs(x.var() - 1) < 5 * np.sqrt(2 / x.size)
    assert stats.kstest(x, "norm").pvalue > 1e-3
    y = x.reshape(8, 25, 200)
    # neighbouring rows / sweeps / chains uncorrelated
    for a, b in ((y[:, :, 1:], y[:, :, :-1]), (y[:, 1:], y[:, :-1]), (y[1:], y[:-1])):
        r = np.corrcoef(a.ravel(), b.ravel())[0, 1]
        assert abs(r) < 5 / np.sqrt(a.size)
    # the two chains of one Box-Muller pair (R4) are independent, not merely uncorrelated:
    # their squares (which share the radius) are uncorrelated too
    r2 = np.corrcoef((y[0::2] ** 2).ravel(), (y[1::2] ** 2).ravel())[0, 1]
    assert abs(r2) < 5 / np.sqrt(y[0::2].size)


# ---------------------------------------------------------- sweep structure

def _split(a):
    D = np.diag(np.diag(a))
    return D, np.tril(a, -1), np.triu(a, 1)


def _gs_iterates(a, z0, w0, k):
    """Textbook Gauss-Seidel on C z = 0 and C^dagger w = 0 (Eq. 12)."""
    D, L, U = _split(a)
    z, w, zs, ws = z0.copy(), w0.copy(), [], []
    for _ in range(k):
        z = sla.solve_triangular(D + L, -U @ z, lower=True)
        w = sla.solve_triangular((D + U).conj().T, -(L.conj().T) @ w, lower=True)
        zs.append(z)
        ws.append(w)
    return np.array(zs), np.array(ws)


def _normwise(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


@pytest.mark.parametrize("cplx", [False, True])
def test_zero_noise_is_gauss_seidel(orc, cplx):
    c = W.random_dense(12, seed=11, complex_=cplx, ratio=0.7)
    a = c.to_dense()
    rng = np.random.default_rng(3)
    z0 = rng.standard_normal(12) + (1j * rng.standard_normal(12) if cplx else 0)
    w0 = rng.standard_normal(12) + (1j * rng.standard_normal(12) if cplx else 0)
    m = orc.Matrix(c)
    r = m.run(seed=1, chains=1, burn_in=6, cycles=0, noise=orc.NOISE_ZERO, z_init=z0, w_init=w0,
              snap_sweeps=range(6))
    zs, ws = _gs_iterates(a, z0, w0, 6)
    assert _normwise(r["z_snap"][:, 0], zs) < 1e-12
    assert _normwise(r["w_snap"][:, 0], ws) < 1e-12


def test_hand_unrolled_n3(orc):
    """SPEC S:186 [DERIVED]: Eq. (4)/(5) evaluated by hand for one sweep,
    phi = 1, zero start. Non-symmetric so a transposed operand fails."""
    a = np.array([[2.0, 0.5, 0.0], [1.0, 4.0, -1.0], [0.25, 2.0, 8.0]])
    m = orc.Matrix(W.CSR.from_dense(a))
    r = m.run(seed=0, chains=1, burn_in=1, cycles=0, noise=orc.NOISE_ONE)
    z0 = 1 / np.sqrt(2)
    z1 = 1 / 2 - (1 / 4) * (1.0 * z0)
    z2 = 1 / np.sqrt(8) - (1 / 8) * (0.25 * z0 + 2.0 * z1)
    w0 = 1 / np.sqrt(2)
    w1 = 1 / 2 - (1 / 4) * (0.5 * w0)
    w2 = 1 / np.sqrt(8) - (1 / 8) * (-1.0 * w1)
    np.testing.assert_allclose(r["z"][0], [z0, z1, z2], rtol=1e-15)
    np.testing.assert_allclose(r["w"][0], [w0, w1, w2], rtol=1e-15)
    # second sweep: old values of later rows enter
    r2 = m.run(seed=0, chains=1, burn_in=2, cycles=0, noise=orc.NOISE_ONE)
    z0b = 1 / np.sqrt(2) - (1 / 2) * (0.5 * z1)
    w0b = 1 / np.sqrt(2) - (1 / 2) * (1.0 * w1 + 0.25 * w2)
    assert r2["z"][0][0] == pytest.approx(z0b, rel=1e-15)
    assert r2["w"][0][0] == pytest.approx(w0b, rel=1e-15)


def test_identity_phi_one(orc):
    """C = I, phi = 1 -> z = w = 1."""
    m = orc.Matrix(W.diagonal(np.ones(5)))
    r = m.run(seed=0, chains=2, burn_in=3, cycles=0, noise=orc.NOISE_ONE)
    assert np.all(r["z"] == 1.0) and np.all(r["w"] == 1.0)


def test_diagonal_closed_form_and_branch(orc):
    """diagonal C gives z_i = phi_i / sqrt(c_ii) after one sweep.
    With diagonals on and off the negative real axis, z_i conj(w_i) must equal
    phi^2 / c_ii (reading R1 / finding F1: w uses conj(1/sqrt(c_ii)))."""
    d = np.array([-2.0 + 0j, -0.5 + 0j, 3.0 + 0j, 1j, -1 - 1e-3j, 2 - 3j], dtype=np.complex128)
    m = orc.Matrix(W.diagonal(d))
    seed = 99
    r = m.run(seed=seed, chains=3, burn_in=1, cycles=0, chain_begin=5)
    for c in range(3):
        phi = np.array([orc.gaussian(seed, i, 0, 5 + c) for i in range(d.size)])
        np.testing.assert_allclose(r["z"][c], phi / np.sqrt(d), rtol=1e-15, atol=0)
        np.testing.assert_allclose(r["z"][c] * np.conj(r["w"][c]), phi**2 / d, rtol=1e-14)
    # statistically: E(z_i conj w_i) = 1/c_ii
    r = m.run(seed=seed, chains=512, burn_in=0, cycles=40, outputs=("diag",))
    est, se = orc.estimate(r["diag"], 40, group_size=1)
    _stats.check(est, 1 / d, se, G=512, what="diag of diagonal C")


@pytest.mark.parametrize("cplx", [False, True])
def test_hermitian_collapse(orc, cplx):
    """for hermitian C (real positive diagonal) w == z exactly."""
    c = W.random_dense(10, seed=5, complex_=cplx, hermitian=True, ratio=0.8)
    m = orc.Matrix(c)
    r = m.run(seed=123, chains=4, burn_in=2, cycles=0, snap_sweeps=[0, 1])
    assert np.array_equal(r["z"], r["w"])
    assert np.array_equal(r["z_snap"], r["w_snap"])
    # ... and a non-hermitian C does not collapse
    c2 = W.random_dense(10, seed=5, complex_=cplx, ratio=0.8)
    r2 = orc.Matrix(c2).run(seed=123, chains=1, burn_in=2, cycles=0)
    assert not np.allclose(r2["z"], r2["w"])


@pytest.mark.parametrize("cplx", [False, True])
def test_coupling_identity(orc, cplx):
    """Eq. (12): two starts sharing the noise differ by a
    Gauss-Seidel iterate of C (z2 - z1) = 0 and C^dagger (w2 - w1) = 0."""
    c = W.random_dense(9, seed=8, complex_=cplx, ratio=0.6)
    a = c.to_dense()
    m = orc.Matrix(c)
    z1 = np.zeros(9, complex if cplx else float)
    z2 = np.arange(9, dtype=float) + (0.5j if cplx else 0)   # Alg. 1 step 1: z* = i
    ra = m.run(seed=4, chains=1, burn_in=3, cycles=0, z_init=z1, w_init=z1, snap_sweeps=[0, 1, 2])
    rb = m.run(seed=4, chains=1, burn_in=3, cycles=0, z_init=z2, w_init=z2, snap_sweeps=[0, 1, 2])
    zs, ws = _gs_iterates(a, z2 - z1, z2 - z1, 3)
    assert _normwise(rb["z_snap"][:, 0] - ra["z_snap"][:, 0], zs) < 1e-12
    assert _normwise(rb["w_snap"][:, 0] - ra["w_snap"][:, 0], ws) < 1e-12


def test_stationary_identity_dense():
    """Eq. (recursive): C^-1 = (D+L)^-1 D (D+U)^-1 + T C^-1 S, with
    T = (D+L)^-1 U, S = L (D+U)^-1; the basis of the
    expectation pins below."""
    for cplx in (False, True):
        for seed in range(20):
            a = W.random_dense(10, seed=seed, complex_=cplx, ratio=0.9).to_dense()
            D, L, U = _split(a)
            T = np.linalg.solve(D + L, U)
            S = L @ np.linalg.inv(D + U)
            Ci = np.linalg.inv(a)
            rhs = np.linalg.solve(D + L, D) @ np.linalg.inv(D + U) + T @ Ci @ S
            assert _normwise(rhs, Ci) < 1e-12


# ------------------------------------------------------------- expectation

def _expected_mean(a, burn_in, cycles):
    """E[estimate] from a zero start: P_0 = 0, P_k = T P_{k-1} S + G with
    G = (D+L)^-1 D (D+U)^-1; the state after sweep s is P_{s+1}, so the
    estimate averages P_{N+1} .. P_{N+M'} (derived from Eq. zk/wk)."""
    D, L, U = _split(a)
    T = np.linalg.solve(D + L, U)
    S = L @ np.linalg.inv(D + U)
    G = np.linalg.solve(D + L, D) @ np.linalg.inv(D + U)
    P = np.zeros_like(G)
    acc = np.zeros_like(G)
    for s in range(burn_in + cycles):
        P = T @ P @ S + G
        if s >= burn_in:
            acc += P
    return acc / cycles


@pytest.mark.parametrize("cplx", [False, True])
def test_exact_finite_k_expectation(orc, cplx):
    """Short runs from z = w = 0 with no burn-in are biased; the oracle's
    estimate must match the exact finite-k mean and must NOT match C^-1
    (so a burn-in or sweep-index slip is caught)."""
    rng = np.random.default_rng(21)
    b = rng.random((5, 5)) * (np.exp(1j * rng.uniform(0, 0.5, (5, 5))) if cplx else 1.0)
    np.fill_diagonal(b, 0)
    d = 1 + rng.random(5)
    a = -b * (0.9 * d / np.abs(b).sum(1))[:, None] + np.diag(d)   # sp(T) close to 0.9
    c = W.CSR.from_dense(a)
    m = orc.Matrix(c)
    chains = 4000
    r = m.run(seed=77, chains=chains, burn_in=1, cycles=2, outputs=("full",))
    est, se = orc.estimate(r["full"], 2, group_size=20)
    G = chains // 20
    _stats.check(est, _expected_mean(a, 1, 2), se, G=G, what="finite-k mean")
    z = _stats.zscores(est, np.linalg.inv(a), se)
    assert np.max(np.abs(z)) > 8, "bias vs C^-1 not visible; test is not discriminating"


@pytest.mark.parametrize("cplx,diag_phase", [(False, None), (True, None), (True, np.pi)])
def test_dense_lu_statistics(orc, cplx, diag_phase):
    """Eq. (1/C): full estimate vs numpy.linalg.inv. The
    diag_phase = pi case puts c_ii on the negative real axis (finding F1)."""
    c = W.random_dense(8, seed=31, complex_=cplx, ratio=0.6, diag_phase=diag_phase)
    a = c.to_dense()
    m = orc.Matrix(c)
    r = m.run(seed=1, chains=256, burn_in=40, cycles=200, outputs=("full", "diag"))
    est, se = orc.estimate(r["full"], 200, group_size=1)
    exact = np.linalg.inv(a)
    _stats.check(est, exact, se, G=256, what="full")
    estd, sed = orc.estimate(r["diag"], 200, group_size=1)
    np.testing.assert_allclose(estd, np.diag(est), rtol=1e-12)
    # the stationary expectation equals C^-1 up to the burn-in bias
    assert _normwise(_expected_mean(a, 40, 200), exact) < 1e-10


def test_pattern_and_config1_shape(orc):
    """Selected elements (pattern) equal the matching full-output entries and
    estimate C^-1 (config-1-like dense matrix at reduced size)."""
    c = W.dense_config1(16, seed=1001)
    a = c.to_dense()
    rows = np.array([0, 3, 15, 7, 7], np.int32)
    cols = np.array([0, 9, 2, 7, 8], np.int32)
    m = orc.Matrix(c, pattern=(rows, cols))
    r = m.run(seed=1, chains=64, burn_in=100, cycles=200, outputs=("full", "pattern"))
    np.testing.assert_allclose(r["pattern"], r["full"][:, rows, cols], rtol=1e-13)
    est, se = orc.estimate(r["pattern"], 200, group_size=1)
    _stats.check(est, np.linalg.inv(a)[rows, cols], se, G=64, what="pattern")


def test_error_falls_as_inverse_sqrt_samples(orc):
    """BASELINE north_star: error falling as 1/sqrt(samples); slope of
    log ||err||_F vs log(chains) in [-0.6, -0.4], averaged over seeds."""
    c = W.random_dense(6, seed=41, ratio=0.6)
    a = c.to_dense()
    exact = np.linalg.inv(a)
    m = orc.Matrix(c)
    ns = [16, 64, 256, 1024]
    errs = []
    for ch in ns:
        e = []
        for s in range(6):
            r = m.run(seed=1000 + s, chains=ch, burn_in=30, cycles=20, outputs=("full",),
                      chain_begin=100000 * s)
            e.append(np.linalg.norm(r["full"].sum(0) / (ch * 20) - exact) ** 2)
        errs.append(np.sqrt(np.mean(e)))
    slope = np.polyfit(np.log(ns), np.log(errs), 1)[0]
    assert -0.6 < slope < -0.4, slope


def test_trace_estimator_w_dagger_q_z(orc):
    """Eq. (tr), reading R2 / finding F2: the oracle's w^dagger Q z
    estimates tr(Q C^-1); the printed z^dagger Q w would estimate
    conj(tr(Q^dagger C^-1)), which differs for this non-hermitian Q."""
    c = W.random_dense(6, seed=51, complex_=True, ratio=0.6)
    q = W.random_q(6, seed=52, per_row=3)
    a, qd = c.to_dense(), q.to_dense()
    m = orc.Matrix(c, q=q)
    r = m.run(seed=9, chains=512, burn_in=40, cycles=100, outputs=("trace",))
    est, se = orc.estimate(r["trace"], 100, group_size=4)
    good = np.trace(qd @ np.linalg.inv(a))
    bad = np.conj(np.trace(qd.conj().T @ np.linalg.inv(a)))
    _stats.check(np.array([est]), np.array([good]), np.array([se]), G=128, what="trace")
    zb = _stats.zscores(np.array([est]), np.array([bad]), np.array([se]))
    assert np.max(np.abs(zb)) > 10


def test_one_draw_gs_agrees_for_hermitian_pd(orc):
    """for hermitian positive-definite C, CC agrees with
    the one-draw Gibbs sampler of Eq. (2), here an independent numpy sampler
    with numpy's own normal noise."""
    c = W.random_dense(6, seed=61, complex_=True, hermitian=True, ratio=0.8)
    a = c.to_dense()
    m = orc.Matrix(c)
    chains, cyc = 400, 100
    r = m.run(seed=3, chains=chains, burn_in=30, cycles=cyc, outputs=("full",))
    est_cc, se_cc = orc.estimate(r["full"], cyc, group_size=4)
    rng = np.random.default_rng(17)
    z = np.zeros((chains, 6), complex)
    acc = np.zeros((chains, 6, 6), complex)
    for k in range(30 + cyc):
        for i in range(6):
            s = z @ a[i] - z[:, i] * a[i, i]
            z[:, i] = rng.standard_normal(chains) / np.sqrt(a[i, i]) - s / a[i, i]
        if k >= 30:
            acc += z[:, :, None] * z[:, None, :].conj()
    g = acc.reshape(chains // 4, 4, 6, 6).sum(1) / (4 * cyc)
    est_gs = g.mean(0)
    se_gs = (g.real.std(0, ddof=1) + 1j * g.imag.std(0, ddof=1)) / np.sqrt(g.shape[0])
    se = np.sqrt(se_cc.real**2 + se_gs.real**2) + 1j * np.sqrt(se_cc.imag**2 + se_gs.imag**2)
    _stats.check(est_cc, est_gs, se, G=100, what="CC vs one-draw GS")
    _stats.check(est_gs, np.linalg.inv(a), se_gs, G=100, what="one-draw GS vs LU")


def test_standard_error_calibration(orc):
    """Mirrors P:558-563 (Geyer SE 0.499 vs 100-replicate empirical 0.502):
    across 40 seeds the spread of the estimates matches the mean group SE."""
    c = W.random_dense(6, seed=71, ratio=0.7)
    m = orc.Matrix(c)
    ests, ses = [], []
    for s in range(40):
        r = m.run(seed=500 + s, chains=64, burn_in=30, cycles=50, outputs=("diag",))
        e, se = orc.estimate(r["diag"], 50, group_size=4)
        ests.append(e)
        ses.append(se)
    ratio = np.std(ests, axis=0, ddof=1) / np.mean(ses, axis=0)
    assert np.all((ratio > 0.6) & (ratio < 1.5)), ratio
    assert 0.8 < np.mean(ratio) < 1.2


def test_pure_gauge_lattice_closed_form(orc):
    """Finding F4: pure-gauge U(1) lattice, diag(C^-1) is the free-field
    constant (1/n) sum_p 1/lambda(p) at every site."""
    c = W.lattice(4, 2, 0.2, seed=5, pure_gauge=True)
    a = c.to_dense()
    val = W.lattice_pure_gauge_diag(4, 2, 0.2)
    np.testing.assert_allclose(np.diag(np.linalg.inv(a)), val, rtol=1e-13)
    m = orc.Matrix(c)
    r = m.run(seed=11, chains=256, burn_in=40, cycles=100, outputs=("diag",))
    est, se = orc.estimate(r["diag"], 100, group_size=2)
    _stats.check(est, np.full(16, val, complex), se, G=128, what="lattice diag")


def test_config_constants_f4():
    """SURVEY F4 full-size closed forms used by the GPU statistical tests."""
    assert W.lattice_pure_gauge_diag(64, 2, 0.2) == pytest.approx(1.124641956079403, rel=1e-13)
    assert W.lattice_pure_gauge_diag(16, 4, 0.1) == pytest.approx(1.055485534357617, rel=1e-13)


# ------------------------------------------------------------- bookkeeping

def test_resume_and_chain_subset(orc):
    """Noise is keyed by absolute (chain, sweep, row): a run split at sweep 4
    and resumed, or a subset of chains run alone, reproduces the same bits."""
    c = W.random_dense(7, seed=81, complex_=True, ratio=0.7)
    m = orc.Matrix(c)
    full = m.run(seed=5, chains=6, burn_in=10, cycles=0)
    part = m.run(seed=5, chains=6, burn_in=4, cycles=0)
    rest = m.run(seed=5, chains=6, burn_in=6, cycles=0, sweep_begin=4, z_init=part["z"], w_init=part["w"])
    assert np.array_equal(full["z"], rest["z"]) and np.array_equal(full["w"], rest["w"])
    sub = m.run(seed=5, chains=2, burn_in=10, cycles=0, chain_begin=3)
    assert np.array_equal(sub["z"], full["z"][3:5])


def test_duplicates_summed(orc):
    a = W.random_dense(5, seed=91, ratio=0.5).to_dense()
    c = W.CSR.from_dense(a)
    # split every entry into two halves, shuffled within each row
    rp, col, val = [0], [], []
    for i in range(5):
        cs = c.col[c.row_ptr[i]:c.row_ptr[i + 1]]
        vs = c.val[c.row_ptr[i]:c.row_ptr[i + 1]]
        cc = np.concatenate([cs, cs])[::-1]
        vv = np.concatenate([vs / 2, vs / 2])[::-1]
        col += list(cc)
        val += list(vv)
        rp.append(len(col))
    dup = W.CSR(5, np.array(rp, np.int64), np.array(col, np.int32), np.array(val))
    r1 = orc.Matrix(c).run(seed=1, chains=2, burn_in=5, cycles=0)
    r2 = orc.Matrix(dup).run(seed=1, chains=2, burn_in=5, cycles=0)
    np.testing.assert_allclose(r1["z"], r2["z"], rtol=1e-14)


def test_errors(orc):
    """D must be non-singular; sp(T) >= 1 diverges."""
    # zero diagonal
    with pytest.raises(orc.OracleError) as e:
        orc.Matrix(W.CSR.from_dense(np.array([[1.0, 1.0], [1.0, 0.0]]), keep_zeros_on_diag=False))
    assert e.value.code == 2
    # real path with a negative diagonal
    with pytest.raises(orc.OracleError) as e:
        orc.Matrix(W.CSR.from_dense(np.array([[1.0, 0.1], [0.1, -2.0]])))
    assert e.value.code == 3
    # sp(T) = 9 > 1
    m = orc.Matrix(W.CSR.from_dense(np.array([[1.0, 3.0], [3.0, 1.0]])))
    with pytest.raises(orc.OracleError) as e:
        m.run(seed=1, chains=1, burn_in=100, cycles=0)
    assert e.value.code == 4


# ------------------------------------------------------------------ Z2 noise (NEXT-1)

def test_z2_noise_bits_and_moments(orc):
    """Reading R21: phi = +1 / -1 from the top bit of word 0 of
    Philox({row, sweep, chain, 1}) (Philox pinned above); E(phi) = 0,
    E(phi^2) = 1 (Eq. 5a/5b; phi = 2B - 1)."""
    seed = 0x5EED00AA
    for (i, k, c) in [(0, 0, 0), (5, 7, 3), (19999, 2199, 1023), (2**31, 1, 2**32 - 1)]:
        w = orc.philox([i, k, c, 1], [seed & 0xFFFFFFFF, seed >> 32])
        assert orc.z2(seed, i, k, c) == (-1.0 if (w[0] >> 31) else 1.0)
    x = np.array([orc.z2(seed, i, k, c) for c in range(4) for k in range(50) for i in range(250)])
    assert set(np.unique(x)) == {-1.0, 1.0}
    assert abs(x.mean()) < 4 / np.sqrt(x.size)


def test_z2_diagonal_is_exact(orc):
    """P:1044-1048 with Z2 noise: z_i = phi sigma_i, w_i = phi conj(sigma_i), so
    every sample z_i conj(w_i) = phi^2 / c_ii = 1/c_ii exactly: the estimate of
    diag(C^-1) is exact with zero variance (the paper's reason to prefer Z2
    noise)."""
    d = np.array([2.0, 4.0, 0.5, 3.0])
    c = W.diagonal(d)
    r = orc.Matrix(c).run(seed=3, chains=8, burn_in=1, cycles=5, outputs=("diag",), noise=orc.NOISE_Z2)
    est, se = orc.estimate(r["diag"], 5, group_size=2)
    # every sample is the same number fl(sigma_i)^2: zero spread, the value 1/c_ii up to rounding
    assert np.allclose(est, 1.0 / d, rtol=1e-15, atol=0) and np.all(se == 0)


def test_z2_dense_lu_statistics(orc):
    """Eq. (1/C) with Z2 noise (E(phi phi^T) = I) converges to the dense-LU
    inverse: aggregate 4-SE rule (reading R14)."""
    from tests import _stats
    c = W.random_dense(10, seed=41)
    inv = np.linalg.inv(c.to_dense())
    r = orc.Matrix(c).run(seed=9, chains=256, burn_in=20, cycles=200, outputs=("full",), noise=orc.NOISE_Z2)
    est, se = orc.estimate(r["full"], 200, group_size=8)
    _stats.check(est.ravel(), inv.ravel(), se.ravel(), G=32, what="z2 full")


# ------------------------------------------------------------------ NEXT-2: coupled burn-in (Alg. 1)

def gs_difference_sweeps(c, tol, max_sweeps=10000):
    """Plain Gauss-Seidel on C d = 0 and C^dagger d = 0 from d0_i = i + 1
    (numpy, row by row): the first sweep p with max |d| < tol in both."""
    A = c.to_dense()
    n = A.shape[0]
    dz = np.arange(1, n + 1).astype(A.dtype)
    dw = dz.copy()
    Ah = A.conj().T
    for p in range(1, max_sweeps + 1):
        for i in range(n):
            dz[i] = -(A[i, :i] @ dz[:i] + A[i, i + 1:] @ dz[i + 1:]) / A[i, i]
            dw[i] = -(Ah[i, :i] @ dw[:i] + Ah[i, i + 1:] @ dw[i + 1:]) / Ah[i, i]
        if max(np.max(np.abs(dz)), np.max(np.abs(dw))) < tol:
            return p
    raise AssertionError("no convergence")


@pytest.mark.parametrize("cplx", [False, True])
def test_coupled_burn_in_four_chains(orc, cplx):
    """Algorithm 1 steps 1-5 run literally in the oracle: the pair
    (z, w) from 0 and (z*, w*) from i + 1 with the same noise; the first sweep
    where both differences are below tol equals the noise-free Gauss-Seidel
    count of Eq. (12) that mcinv_coupled_burn_in uses (reading R23)."""
    c = W.lattice(4, 2, 0.2, seed=61) if cplx else W.pedigree(60, seed=62)
    tol = 1e-5
    p_gs = gs_difference_sweeps(c, tol)
    m = orc.Matrix(c)
    dt = np.complex128 if cplx else np.float64
    start = np.arange(1, c.n + 1).astype(dt)
    snaps = list(range(p_gs + 2))
    a = m.run(seed=5, chains=1, burn_in=p_gs + 2, cycles=0, snap_sweeps=snaps, chain_begin=3)
    b = m.run(seed=5, chains=1, burn_in=p_gs + 2, cycles=0, snap_sweeps=snaps, chain_begin=3, z_init=start,
              w_init=start)
    first = None
    for k in snaps:
        dz = np.max(np.abs(b["z_snap"][k, 0] - a["z_snap"][k, 0]))
        dw = np.max(np.abs(b["w_snap"][k, 0] - a["w_snap"][k, 0]))
        if max(dz, dw) < tol:
            first = k + 1  # snapshot k is taken after sweep k + 1
            break
    assert first == p_gs


# ------------------------------------------------------------------ Geyer ESS (NEXT-2)

def test_geyer_hand_computed(orc):
    """orc_geyer on x = 1, 2, 3, 4 worked by hand: xbar 2.5, gamma = (1.25,
    0.3125, -0.375, -0.5625) (lag sums over m - k terms, divided by m), pair
    sums 1.5625 (kept) and -0.9375 (stop), sigma2 = -1.25 + 2 x 1.5625 = 1.875,
    ESS = 4 x 1.25 / 1.875 = 8/3."""
    g = orc.geyer([1.0, 2.0, 3.0, 4.0])
    assert g["mean"] == 2.5 and g["gamma0"] == 1.25
    assert g["sigma2"] == pytest.approx(1.875, rel=1e-15)
    assert g["ess"] == pytest.approx(8 / 3, rel=1e-15)
    assert g["se"] == pytest.approx(np.sqrt(1.875 / 4), rel=1e-15)


@pytest.mark.parametrize("rho", [0.0, 0.9, -0.5])
def test_geyer_ar1_closed_form(orc, rho):
    """AR(1) x_t = rho x_{t-1} + e_t: the integrated autocorrelation time is
    (1 + rho) / (1 - rho), so ESS / m -> (1 - rho) / (1 + rho) (Geyer 1992,
    the estimator of P:354-360); a long series lands within a few percent."""
    rng = np.random.default_rng(31)
    m = 400000
    e = rng.standard_normal(m)
    x = np.empty(m)
    x[0] = e[0] / np.sqrt(1 - rho * rho)
    for t in range(1, m):
        x[t] = rho * x[t - 1] + e[t]
    g = orc.geyer(x)
    want = (1 - rho) / (1 + rho)
    assert g["ess"] / m == pytest.approx(want, rel=0.08)
    assert g["se"] == pytest.approx(np.sqrt(g["gamma0"] / g["ess"]), rel=1e-12)


def test_geyer_identity_matches_the_papers_tables(orc):
    """The paper's standard errors are sqrt(Var / Eff. length) (Table 2,
    P:618-648: 3932 / 15788 -> 0.499, 8123 / 8163 -> 0.998; Table 4,
    P:898-924): the same identity orc_geyer's se = sqrt(gamma_0 / ESS) obeys."""
    for var, ess, se in ((3932.0, 15788.0, 0.499), (8123.0, 8163.0, 0.998)):
        assert np.sqrt(var / ess) == pytest.approx(se, abs=6e-4)
    g = orc.geyer(np.sin(np.arange(5000) * 0.37) + np.random.default_rng(2).standard_normal(5000))
    assert g["se"] == pytest.approx(np.sqrt(g["gamma0"] / g["ess"]), rel=1e-12)


def test_trace_series_sums_to_the_trace(orc):
    """The per-sweep realized traces (Geyer's series) of a run add up to the
    per-chain trace sums, and their mean is the Eq. (tr) estimate."""
    c = W.lattice(3, 2, 0.2, seed=35)
    q = W.random_q(c.n, 36, 2)
    r = orc.Matrix(c, q=q).run(5, 6, 3, 40, ("trace",))
    assert r["trace_series"].shape == (40,)
    assert r["trace_series"].sum() == pytest.approx(r["trace"].sum(), rel=1e-12)
    est, _ = orc.estimate(r["trace"], 40, group_size=6)
    assert r["trace_series"].mean() / 6 == pytest.approx(est, rel=1e-12)
