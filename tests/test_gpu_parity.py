"""GPU (CUDA path through the C ABI) vs oracle, same seeds -- the parity gate.

Levels (BASELINE.json north_star):
  1. Philox words bit-exact; Gaussian within 1e-15 relative.
  2. post-sweep z, w within 1e-12 normwise relative error per chain.
  3. estimates within 1e-10 relative Frobenius and normwise max error.
Sizes: every BASELINE config at a reduced size that spans several warps /
groups and a ragged tail, plus full-size runs compared on sampled chains
(state after all sweeps) and on exact properties (deterministic solves,
pure-gauge closed form).
"""
import numpy as np
import pytest

import workloads as W
from tests import _stats

pytestmark = pytest.mark.gpu

TOL_STATE = 1e-12
TOL_EST = 1e-10


@pytest.fixture(scope="module")
def mc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0412107_b200 as M
    M.load()
    return M


def normwise(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den > 0 else 1.0)


def frob(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def states_match(zg, wg, zo, wo, tol=TOL_STATE):
    for c in range(zo.shape[0]):
        assert normwise(zg[c], zo[c]) < tol, f"z chain {c}: {normwise(zg[c], zo[c])}"
        assert normwise(wg[c], wo[c]) < tol, f"w chain {c}: {normwise(wg[c], wo[c])}"


def est_match(eg, eo, tol=TOL_EST, what=""):
    assert normwise(eg, eo) < tol, f"{what} normwise {normwise(eg, eo)}"
    assert frob(eg, eo) < tol, f"{what} frobenius {frob(eg, eo)}"


def compare_run(mc, orc, c, q=None, pattern=None, seed=1, chains=64, burn_in=5, cycles=10, outputs=("diag",),
                group_size=32, chain_begin=0, snapshot_sweeps=0, noise="gauss"):
    inv = mc.Inverter(c, q=q, pattern=pattern)
    inv.run(seed, chains, burn_in, cycles, outputs, chain_begin=chain_begin, group_size=group_size,
            snapshot_sweeps=snapshot_sweeps, noise=noise)
    res = {o: inv.result(o) for o in outputs}
    zg, wg = inv.get_state()
    om = orc.Matrix(c, q=q, pattern=pattern if pattern is not None else
                    (np.repeat(np.arange(c.n), np.diff(c.row_ptr)).astype(np.int32), c.col))
    r = om.run(seed, chains, burn_in, cycles, outputs, chain_begin=chain_begin,
               noise={"gauss": orc.NOISE_GAUSS, "z2": orc.NOISE_Z2}[noise])
    states_match(zg, wg, r["z"], r["w"])
    for o in outputs:
        eo, so = orc.estimate(r[o], cycles, group_size=group_size, chain_begin=chain_begin)
        eg, sg = res[o]
        est_match(eg, eo, what=o)
        if chains // group_size >= 2:
            # both two-pass about the groups' mean (GPU: moments_kernel; oracle: np.std); they
            # differ only by the summation order of the group sums (atomics)
            assert normwise(sg, so) < 1e-10, f"{o} SE {normwise(sg, so)}"
    inv.close()
    return res


# ------------------------------------------------------------- level 1

def test_philox_bit_exact(mc, orc):
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, size=(2000, 4), dtype=np.uint64).astype(np.uint32)
    ctr[:10] = [[0, 0, 0, 0]] * 10
    ctr[10] = [0xFFFFFFFF] * 4
    for seed in (0, 0x5EED0002, 2**64 - 1, 0x123456789ABCDEF):
        g = mc.philox(ctr, seed)
        for k in range(0, 2000, 7):
            assert list(g[k]) == list(orc.philox(ctr[k], [seed & 0xFFFFFFFF, seed >> 32])), (seed, k)


def test_gaussian_matches_oracle(mc, orc):
    rng = np.random.default_rng(1)
    ctr = np.stack([rng.integers(0, 20000, 3000), rng.integers(0, 2200, 3000), rng.integers(0, 1024, 3000),
                    np.zeros(3000, int)], 1).astype(np.uint32)
    seed = 0x5EED0002
    g = mc.gaussian(ctr, seed)
    o = np.array([orc.gaussian(seed, int(a), int(b), int(c)) for a, b, c, _ in ctr])
    assert np.max(np.abs(g - o) / np.maximum(np.abs(o), 1e-3)) < 1e-15 * 16


# ------------------------------------------------------------- level 2/3, reduced sizes

def test_config1_full_parity(mc, orc):
    """Config 1 exactly as BASELINE.json states it: n=64 dense real, 64 chains,
    100 burn-in + 1000 cycles, full C^-1 (group_size 1 -> G = 64)."""
    c, _, run = W.config(1)
    res = compare_run(mc, orc, c, seed=run.seed, chains=run.chains, burn_in=run.burn_in, cycles=run.cycles,
                      outputs=("full",), group_size=run.group_size)
    est, se = res["full"]
    _stats.check(est, np.linalg.inv(c.to_dense()), se, G=64, what="config1 full vs LU")


def test_config2_reduced_parity(mc, orc):
    """Pedigree matrix (config 2 recipe) at n=3000, 72 chains (ragged last
    warp), diag + pattern with groups of 8."""
    c = W.pedigree(3000, seed=1002)
    compare_run(mc, orc, c, seed=0x5EED0002, chains=72, burn_in=4, cycles=6, outputs=("diag", "pattern"),
                group_size=8)


def test_config3_reduced_parity(mc, orc):
    """Complex lattice (config 3 recipe) at L=8, full output through the DMMA
    contraction, several snapshot chunks (T=4) and a ragged chunk."""
    c = W.lattice(8, 2, 0.2, seed=1003)
    compare_run(mc, orc, c, seed=0x5EED0003, chains=96, burn_in=3, cycles=10, outputs=("full", "diag"),
                group_size=16, snapshot_sweeps=4)


def test_config3_real_full_gemm_tiles(mc, orc):
    """Real full output with n=100 (ragged 64x64 tiles) and group size 4."""
    c = W.random_dense(100, seed=9, ratio=0.5, density=0.2)
    compare_run(mc, orc, c, seed=3, chains=32, burn_in=2, cycles=7, outputs=("full",), group_size=4,
                snapshot_sweeps=3)


def test_config5_reduced_parity(mc, orc):
    """4-D complex lattice (config 5 recipe) at 4^4 with Q (4 nnz/row):
    diag + trace (w^dagger Q z, reading R2)."""
    c = W.lattice(4, 4, 0.1, seed=1005)
    q = W.random_q(c.n, 2005, 4)
    compare_run(mc, orc, c, q=q, seed=0x5EED0005, chains=64, burn_in=3, cycles=8, outputs=("diag", "trace"),
                group_size=32)


def test_all_outputs_complex_nonhermitian(mc, orc):
    c = W.random_dense(40, seed=12, complex_=True, ratio=0.6, density=0.3, diag_phase=np.pi)
    q = W.random_q(40, 13, 3)
    rows = np.array([0, 5, 39, 12, 12, 7], np.int32)
    cols = np.array([0, 30, 2, 12, 13, 7], np.int32)
    compare_run(mc, orc, c, q=q, pattern=(rows, cols), seed=77, chains=40, burn_in=2, cycles=5,
                outputs=("diag", "pattern", "full", "trace"), group_size=8, snapshot_sweeps=2)


def test_nonsymmetric_structure(mc, orc):
    """Row i and column i with different patterns (union lists with zeros)."""
    a = np.triu(W.random_dense(30, seed=14, ratio=0.5).to_dense())  # upper triangle only
    a[np.arange(1, 30), np.arange(29)] = -0.1                         # plus a sub-diagonal
    c = W.CSR.from_dense(a)
    compare_run(mc, orc, c, seed=5, chains=32, burn_in=3, cycles=4, outputs=("diag", "pattern"), group_size=2)


def test_zero_noise_gauss_seidel(mc, orc):
    """noise = zero from a non-zero start reproduces the oracle's GS iterates."""
    c = W.random_dense(50, seed=15, complex_=True, ratio=0.7, density=0.2)
    inv = mc.Inverter(c)
    inv.run(1, 32, 0, 0, ("diag",), group_size=32, noise="zero")
    rng = np.random.default_rng(2)
    z0 = rng.standard_normal((32, 50)) + 1j * rng.standard_normal((32, 50))
    w0 = rng.standard_normal((32, 50)) + 1j * rng.standard_normal((32, 50))
    inv.set_state(z0, w0)
    inv.run(1, 32, 5, 0, ("diag",), group_size=32, noise="zero", resume=True)
    zg, wg = inv.get_state()
    r = orc.Matrix(c).run(1, 32, 5, 0, noise=orc.NOISE_ZERO, z_init=z0, w_init=w0)
    states_match(zg, wg, r["z"], r["w"])


def test_edge_cases(mc, orc):
    # n = 1
    compare_run(mc, orc, W.diagonal(np.array([2.5])), seed=1, chains=32, burn_in=1, cycles=3,
                outputs=("diag", "full"), group_size=4)
    # diagonal complex with the branch cut
    compare_run(mc, orc, W.diagonal(np.array([-2.0 + 0j, 1j, 3.0, -1 - 1e-3j])), seed=2, chains=33 * 1,
                burn_in=0, cycles=4, outputs=("diag",), group_size=1)
    # burn-in only (cycles = 0): no estimate yet (E_STATE); resuming with cycles gives the
    # same result as one run with the burn-in and the cycles (exact resume)
    c2 = W.pedigree(200, seed=4)
    inv = mc.Inverter(c2)
    inv.run(5, 64, 3, 0, ("diag",), group_size=8)
    with pytest.raises(mc.MCInvError) as e:
        inv.result("diag")
    assert e.value.code == 8
    inv.run(5, 64, 0, 4, ("diag",), group_size=8, sweep_begin=3, resume=True)
    e1, _ = inv.result("diag")
    inv.close()
    one = mc.Inverter(c2)
    one.run(5, 64, 3, 4, ("diag",), group_size=8)
    e2, _ = one.result("diag")
    one.close()
    np.testing.assert_allclose(e1, e2, rtol=1e-12, atol=0)  # atomics: summation order may differ
    # empty pattern list
    c = W.random_dense(8, seed=3)
    inv = mc.Inverter(c, pattern=(np.zeros(0, np.int32), np.zeros(0, np.int32)))
    inv.run(1, 32, 1, 2, ("pattern", "diag"))
    e, s = inv.result("pattern")
    assert e.size == 0
    inv.close()


def test_sharding_invariance_and_resume(mc):
    """Chains keyed by global index: two shards summed == one run (moments),
    and a run split in two sweeps ranges == one run (bitwise state)."""
    c = W.pedigree(2000, seed=7)
    a = mc.Inverter(c)
    a.run(9, 128, 3, 5, ("diag", "pattern"), group_size=32)
    full = a.accumulators().cpu().numpy().copy()
    z_all, w_all = a.get_state()
    b = mc.Inverter(c)
    parts = []
    for cb in (0, 64):
        b.run(9, 64, 3, 5, ("diag", "pattern"), chain_begin=cb, group_size=32)
        parts.append(b.accumulators().cpu().numpy().copy())
        zb, wb = b.get_state()
        assert np.array_equal(zb, z_all[cb:cb + 64]) and np.array_equal(wb, w_all[cb:cb + 64])
    nS1 = (full.size - 1) // 2  # [S1 | M2 | divergence]: the S1 blocks of the shards add up
    np.testing.assert_allclose(parts[0][:nS1] + parts[1][:nS1], full[:nS1], rtol=1e-12, atol=1e-300)
    # resume: 8 sweeps == 3 + 5
    b.run(9, 128, 3, 0, ("diag",), group_size=32)
    b.run(9, 128, 0, 5, ("diag",), group_size=32, sweep_begin=3, resume=True)
    zr, wr = b.get_state()
    a.run(9, 128, 8, 0, ("diag",), group_size=32)
    z8, w8 = a.get_state()
    assert np.array_equal(zr, z8) and np.array_equal(wr, w8)


def test_errors(mc):
    M = mc
    with pytest.raises(M.MCInvError) as e:
        M.Inverter(W.CSR.from_dense(np.array([[1.0, 1.0], [1.0, 0.0]]), keep_zeros_on_diag=False))
    assert e.value.code == 2 and e.value.index == 1
    with pytest.raises(M.MCInvError) as e:
        M.Inverter(W.CSR.from_dense(np.array([[1.0, 0.1], [0.1, -2.0]])))
    assert e.value.code == 3
    inv = M.Inverter(W.CSR.from_dense(np.array([[1.0, 3.0], [3.0, 1.0]])))  # sp(T) = 9
    inv.run(1, 32, 200, 1, ("diag",))
    with pytest.raises(M.MCInvError) as e:
        inv.result("diag")
    assert e.value.code == 4
    with pytest.raises(M.MCInvError) as e:
        inv.run(1, 30, 1, 1, ("diag",), group_size=32)  # chains not a multiple of group_size
    assert e.value.code == 1
    with pytest.raises(M.MCInvError) as e:
        inv.run(1, 32, 1, 1, ("trace",))  # no Q
    assert e.value.code == 8


@pytest.mark.parametrize("kernel", ["v1", "v3"])
def test_both_kernels(mc, orc, kernel, monkeypatch):
    """The row-by-row kernel (v1) and the level-scheduled kernel (v3) both
    match the oracle; v3 for every chains-per-CTA layout: C below, equal to
    and above the group size and above a warp."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    Cs = {"v1": (32,), "v3": (1, 4, 8, 32, 64)}[kernel]
    for C in Cs:
        monkeypatch.setenv("MCINV_C", str(C))
        compare_run(mc, orc, W.pedigree(500, seed=21), seed=4, chains=64, burn_in=2, cycles=4,
                    outputs=("diag", "pattern"), group_size=8)
        c = W.lattice(4, 3, 0.15, seed=22)
        compare_run(mc, orc, c, q=W.random_q(c.n, 23, 3), seed=5, chains=40, burn_in=2, cycles=3,
                    outputs=("diag", "trace", "full"), group_size=4, snapshot_sweeps=2)


@pytest.mark.parametrize("kernel", ["v4", "v5"])
def test_v4_dataflow(mc, orc, monkeypatch, kernel):
    """The dataflow kernel (v4: per-row completion counters, no level barriers;
    v5: the same with TMA-staged plan blocks) matches the oracle for every
    chains-per-CTA layout up to a warp, real and complex, with diag / pattern /
    full outputs, several launches (full-output chunks) and forced block
    sizes; the automatic kernel choice is checked at the end."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    for C in (1, 4, 8, 32):
        monkeypatch.setenv("MCINV_C", str(C))
        for th in ("64", "768"):
            monkeypatch.setenv("MCINV_THREADS", th)
            compare_run(mc, orc, W.pedigree(500, seed=21), seed=4, chains=64, burn_in=2, cycles=4,
                        outputs=("diag", "pattern"), group_size=8)
        c = W.lattice(4, 3, 0.15, seed=22)
        compare_run(mc, orc, c, seed=5, chains=40, burn_in=2, cycles=3, outputs=("diag", "full"), group_size=4,
                    snapshot_sweeps=2)
    monkeypatch.delenv("MCINV_KERNEL")
    monkeypatch.delenv("MCINV_C")
    monkeypatch.delenv("MCINV_THREADS")
    # automatic choice: v4 where it applies (configs 2, 3), v3 for C > 32 or trace (configs 4, 5)
    for k, ver in ((3, (4, 5)), (2, (4, 5, 6)), (5, (5,))):
        c, q, run = W.config(k)
        inv = mc.Inverter(c, q=q)
        inv.run(run.seed, run.chains, 0, 1, tuple(o for o in run.outputs if o != "full") or ("diag",),
                group_size=run.group_size)
        assert inv.kernel_info()["version"] in ver, k
        inv.close()


@pytest.mark.parametrize("threads", ["768", "512", "96"])
def test_v5_trace_phase(mc, orc, monkeypatch, threads):
    """v5 with trace items (w^dagger Q z, reading R2) as a phase after every
    sampling sweep: complex and real C, every chains-per-CTA layout up to a
    warp, Gaussian and Z2 noise, the per-sweep series, several launches."""
    monkeypatch.setenv("MCINV_KERNEL", "v5")
    monkeypatch.setenv("MCINV_THREADS", threads)
    c = W.lattice(4, 3, 0.15, seed=81)
    q = W.random_q(c.n, 82, 4)
    p = W.pedigree(500, seed=83)
    qp = W.random_q(p.n, 84, 3, complex_=False)
    for C in (1, 4, 16, 32):
        monkeypatch.setenv("MCINV_C", str(C))
        compare_run(mc, orc, c, q=q, seed=21, chains=64, burn_in=2, cycles=5, outputs=("diag", "trace"),
                    group_size=8)
        compare_run(mc, orc, p, q=qp, seed=22, chains=96, burn_in=3, cycles=4, outputs=("trace", "diag", "pattern"),
                    group_size=16, noise="z2" if C == 4 else "gauss")


@pytest.mark.parametrize("threads", ["512", "768", "1024", "256"])
def test_v6_two_chains_per_thread(mc, orc, monkeypatch, threads):
    """v6 (the dataflow kernel with the two chains of a Box-Muller pair per
    thread, reading R4) for every chains-per-CTA layout C = 2..32 (R = 64/C rows
    per warp item), SE groups smaller than, equal to and larger than C, a
    ragged chain count, an odd-group shard start, and diag / pattern / full."""
    monkeypatch.setenv("MCINV_KERNEL", "v6")
    monkeypatch.setenv("MCINV_THREADS", threads)
    for C, gs, chains, cb in ((2, 2, 62, 0), (4, 4, 68, 4), (8, 32, 96, 32), (8, 2, 64, 6), (16, 8, 48, 0),
                              (32, 32, 64, 64)):
        monkeypatch.setenv("MCINV_C", str(C))
        compare_run(mc, orc, W.pedigree(700, seed=25), seed=13, chains=chains, burn_in=3, cycles=4,
                    outputs=("diag", "pattern"), group_size=gs, chain_begin=cb)
    monkeypatch.setenv("MCINV_C", "8")
    compare_run(mc, orc, W.dense_config1(24, seed=26), seed=14, chains=64, burn_in=1, cycles=3,
                outputs=("diag", "full"), group_size=8, snapshot_sweeps=2)
    for noise in ("z2",):
        compare_run(mc, orc, W.pedigree(300, seed=27), seed=15, chains=64, burn_in=2, cycles=3,
                    outputs=("diag", "pattern"), group_size=16, noise=noise)


@pytest.mark.parametrize("kernel", ["v3", "v4"])
@pytest.mark.parametrize("K", ["1", "2"])
def test_chains_per_thread(mc, orc, monkeypatch, K, kernel):
    """v3 and v4 with one or two adjacent chains per thread (256-bit state
    accesses, in-thread pre-summed accumulation) for several chains-per-CTA
    layouts and group sizes, including an inactive tail chain."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    monkeypatch.setenv("MCINV_K", K)
    for C, gs, chains in ((2, 2, 62), (8, 8, 64), (16, 4, 60)) + (((64, 32, 96),) if kernel == "v3" else ()):
        monkeypatch.setenv("MCINV_C", str(C))
        compare_run(mc, orc, W.pedigree(400, seed=23), seed=7, chains=chains, burn_in=2, cycles=3,
                    outputs=("diag", "pattern"), group_size=gs)
        compare_run(mc, orc, W.dense_config1(24, seed=24), seed=8, chains=chains, burn_in=1, cycles=3,
                    outputs=("diag", "full"), group_size=gs, snapshot_sweeps=2)


@pytest.mark.parametrize("kernel", ["v1", "v3", "v4", "v5"])
def test_z2_noise_parity(mc, orc, kernel, monkeypatch):
    """NEXT-1 Z2 noise (reading R21) on every sweep kernel:
    states and estimates vs the oracle on the same seed."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    compare_run(mc, orc, W.pedigree(400, seed=51), seed=11, chains=64, burn_in=2, cycles=4,
                outputs=("diag", "pattern"), group_size=8, noise="z2")
    c = W.lattice(4, 3, 0.15, seed=52)
    outs = ("diag", "trace") if kernel not in ("v4", "v5") else ("diag", "full")
    compare_run(mc, orc, c, q=W.random_q(c.n, 53, 3) if "trace" in outs else None, seed=12, chains=40, burn_in=2,
                cycles=3, outputs=outs, group_size=4, noise="z2", snapshot_sweeps=2)


def test_v3_custom_pattern_and_threads(mc, orc, monkeypatch):
    """v3 with a custom pattern (non-neighbour pairs, duplicates, diagonal
    elements: deferred items) and forced block sizes (several rounds of items
    per phase)."""
    monkeypatch.setenv("MCINV_KERNEL", "v3")
    c = W.pedigree(300, seed=31)
    rng = np.random.default_rng(32)
    pr = rng.integers(0, c.n, 200).astype(np.int32)
    pc = rng.integers(0, c.n, 200).astype(np.int32)
    pr[:5] = pc[:5]            # diagonal elements
    pr[5:10] = pr[0:5]         # duplicates
    pc[5:10] = pc[0:5]
    for th in ("32", "96", "1024"):
        monkeypatch.setenv("MCINV_THREADS", th)
        compare_run(mc, orc, c, pattern=(pr, pc), seed=6, chains=48, burn_in=1, cycles=3,
                    outputs=("pattern", "diag"), group_size=16)


def test_bench_configs_use_level_kernels(mc):
    for k in (2, 3, 5):
        c, q, run = W.config(k)
        inv = mc.Inverter(c, q=q)
        inv.run(run.seed, run.chains, 0, 1, tuple(o for o in run.outputs if o != "full") or ("diag",),
                group_size=run.group_size)
        assert inv.kernel_info()["version"] in (3, 4, 5, 6), k
        inv.close()


# ------------------------------------------------------------- full sizes (bench launch configuration)

def _exact_columns(c, cols, tol=1e-14):
    """X = C^-1[:, cols] by Jacobi iteration X <- D^-1 (E - (C - D) X); the
    config-2/4 recipe is strictly row diagonally dominant (factor 1.1), so
    ||D^-1 (C - D)||_inf = 1/1.1 and the iteration converges to tol."""
    A = c.to_scipy()
    d = A.diagonal()
    off = A - __import__("scipy.sparse", fromlist=["diags"]).diags(d)
    E = np.zeros((c.n, len(cols)), dtype=c.val.dtype)
    E[cols, np.arange(len(cols))] = 1
    X = E / d[:, None]
    for _ in range(2000):
        Xn = (E - off @ X) / d[:, None]
        if np.max(np.abs(Xn - X)) < tol * np.max(np.abs(Xn)):
            return Xn
        X = Xn
    raise RuntimeError("Jacobi did not converge")


def test_config2_full_size(mc, orc):
    """Config 2 exactly as bench.py times it (n=20000, 1024 chains, 200+2000
    sweeps, diag + pattern): sampled chains' final states vs the oracle, and
    diag / pattern estimates of sampled rows vs exact sparse solves."""
    c, _, run = W.config(2)
    inv = mc.Inverter(c)
    inv.run(run.seed, run.chains, run.burn_in, run.cycles, run.outputs, group_size=run.group_size)
    ed, sd = inv.result("diag")
    ep, sp_ = inv.result("pattern")
    picks = [0, 517, 1023]
    om = orc.Matrix(c)
    for ch in picks:
        r = om.run(run.seed, 1, run.burn_in + run.cycles, 0, chain_begin=ch)
        zg, wg = inv.get_state(ch, 1)
        states_match(zg, wg, r["z"], r["w"])
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(c.n, 60, replace=False))
    X = _exact_columns(c, rows)                    # X[:, k] = C^-1[:, rows[k]]
    exact_d = X[rows, np.arange(len(rows))]
    _stats.check(ed[rows], exact_d, sd[rows], G=32, what="config2 diag")
    # pattern elements (i, j) with j in the sampled columns
    pr = np.repeat(np.arange(c.n), np.diff(c.row_ptr))
    sel = np.isin(c.col, rows)
    pos = {r: k for k, r in enumerate(rows)}
    exact_p = np.array([X[i, pos[j]] for i, j in zip(pr[sel], c.col[sel])])
    _stats.check(ep[sel], exact_p, sp_[sel], G=32, what="config2 pattern")


@pytest.mark.slow
def test_config5_full_size_pure_gauge(mc, orc):
    """Config 5 launch configuration (16^4 complex, 16384 chains, diag +
    trace) on the pure-gauge variant: diag(C^-1) = 1.055485534357617 at every
    site (finding F4); sampled chain states vs the oracle (reduced sweeps)."""
    c, q, run = W.config(5, pure_gauge=True)
    inv = mc.Inverter(c, q=q)
    inv.run(run.seed, run.chains, run.burn_in, run.cycles, run.outputs, group_size=run.group_size)
    ed, sd = inv.result("diag")
    _stats.check(ed, np.full(c.n, 1.055485534357617 + 0j), sd, G=run.chains // 32, what="config5 diag")
    inv.run(run.seed, 64, 3, 0, ("diag",), chain_begin=16384 - 64)
    zg, wg = inv.get_state(60, 4)
    r = orc.Matrix(c).run(run.seed, 4, 3, 0, chain_begin=16384 - 4)
    states_match(zg, wg, r["z"], r["w"])


def test_config4_sampled_sweeps(mc, orc):
    """Config 4 matrix (n = 1e6 pedigree): 2 sweeps of 64 chains, sampled
    chain states vs the oracle."""
    c, _, run = W.config(4)
    inv = mc.Inverter(c)
    inv.run(run.seed, 64, 2, 0, ("diag",), chain_begin=8192 - 64)
    zg, wg = inv.get_state(62, 2)
    r = orc.Matrix(c).run(run.seed, 2, 2, 0, chain_begin=8192 - 2)
    states_match(zg, wg, r["z"], r["w"])


# ------------------------------------------------------------- NEXT-3: free Wilson-Dirac

def test_dirac_parity(mc, orc):
    """Dirac 3^4 lattice (complex non-hermitian, 14 nnz/row): states, diag and
    tr(Q L^-1) with Q = I vs the oracle on the same seed."""
    c = W.dirac(3)
    compare_run(mc, orc, c, q=W.identity_q(c.n), seed=21, chains=64, burn_in=3, cycles=4,
                outputs=("diag", "trace"), group_size=16)


@pytest.mark.slow
@pytest.mark.parametrize("N,printed", [(18, 413007.84), (20, 629489.14)])
def test_dirac_trace_matches_paper(mc, N, printed):
    """The paper's Dirac cases (K = 0.1, Q = I): Tables 3/4, N = 18 (n = 419,904;
    exact value printed 413007.84) and Table 5, N = 20 (n = 640,000;
    printed 629489.14). The GPU estimate of tr(L^-1) agrees with the
    exact value (the closed form, itself pinned to the printed values in
    tests/test_dirac.py) within 4 standard errors (scalar rule, reading R14)."""
    c = W.dirac(N)
    exact = W.dirac_trace_closed(N)
    assert abs(exact - printed) < 0.02
    inv = mc.Inverter(c, q=W.identity_q(c.n))
    inv.run(0x5EED0012 + (N - 18), 2048, 30, 200, ("trace",), group_size=32)
    est, se = inv.result("trace")
    r = (est.real - exact) / se.real
    assert abs(r) < 4, (est, se, exact)
    assert abs(est.imag) < 4 * se.imag + 1e-9
    inv.close()


# ------------------------------------------------------------- NEXT-2: coupled burn-in, adaptive stopping

@pytest.mark.parametrize("cplx", [False, True])
def test_coupled_burn_in_matches_gauss_seidel(mc, cplx):
    """mcinv_coupled_burn_in (Alg. 1 steps 1-5 via Eq. 12) equals the plain
    Gauss-Seidel count on the start difference (which the oracle's literal
    four-chain run also reproduces, test_oracle_pins)."""
    from tests.test_oracle_pins import gs_difference_sweeps
    c = W.lattice(4, 2, 0.2, seed=61) if cplx else W.pedigree(60, seed=62)
    inv = mc.Inverter(c)
    n, d = inv.coupled_burn_in(1e-5)
    assert n == gs_difference_sweeps(c, 1e-5) and d < 1e-5
    inv.close()


def test_run_until_adaptive(mc, orc):
    """Adaptive stopping (mcinv_run_until): blocks of sampling sweeps until the
    relative SE of the trace is below the target; the estimate equals the oracle
    run with the same total sweeps (resume is exact), and the SE target holds."""
    c = W.lattice(3, 2, 0.2, seed=63)
    q = W.identity_q(c.n)
    inv = mc.Inverter(c, q=q)
    burn, _ = inv.coupled_burn_in(1e-6)
    done, rse = inv.run_until(17, 64, burn, ("trace", "diag"), "trace", 2e-3, check_cycles=20, max_cycles=2000,
                              group_size=8)
    assert done % 20 == 0 and rse < 2e-3
    est, se = inv.result("trace")
    assert abs(se) / abs(est) < 2e-3
    r = orc.Matrix(c, q=q).run(17, 64, burn, done, ("trace",))
    eo, so = orc.estimate(r["trace"], done, group_size=8)
    assert abs(est - eo) < 1e-10 * abs(eo)
    inv.close()


@pytest.mark.slow
def test_config3_full_size_dense_lu(mc, orc):
    """Config 3 exactly as specified (BASELINE configs[2]: 64^2 complex lattice,
    2048 chains, 200 + 2000 sweeps, full C^-1 through the DMMA contraction):
    all 16.7M elements vs the dense LU inverse with the aggregate rule of
    reading R14 (G = 64 groups), and sampled chains' final states vs the
    oracle."""
    c, _, run = W.config(3)
    inv = mc.Inverter(c)
    inv.run(run.seed, run.chains, run.burn_in, run.cycles, ("full",), group_size=run.group_size)
    est, se = inv.result("full")
    exact = np.linalg.inv(c.to_dense())
    G = run.chains // run.group_size
    _stats.check(est.real.ravel(), exact.real.ravel(), se.real.ravel(), G=G, what="config3 full re")
    _stats.check(est.imag.ravel(), exact.imag.ravel(), se.imag.ravel(), G=G, what="config3 full im")
    for ch in (0, 2047):
        r = orc.Matrix(c).run(run.seed, 1, run.burn_in + run.cycles, 0, chain_begin=ch)
        zg, wg = inv.get_state(ch, 1)
        states_match(zg, wg, r["z"], r["w"])
    inv.close()


@pytest.mark.parametrize("kernel", ["v1", "v3", "v4", "v5", "v6"])
def test_irregular_structure(mc, orc, kernel, monkeypatch):
    """An unsorted CSR with duplicate entries (summed), explicit zeros (kept),
    rows with no off-diagonal entry and a few dense rows (long entry lists:
    several gather chunks), a non-symmetric pattern, and a shard that starts
    at chain 64: every kernel vs the oracle."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    if kernel == "v6":
        monkeypatch.setenv("MCINV_C", "4")  # v6 holds two chains per thread: C >= 2
    rng = np.random.default_rng(77)
    n = 150
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i), cols.append(i), vals.append(0.0)  # diagonal fixed below
        if i % 7 == 3:
            continue  # diagonal only
        k = 40 if i % 25 == 0 else rng.integers(1, 6)
        for j in rng.choice(n, size=k, replace=False):
            if j != i:
                rows.append(i), cols.append(int(j)), vals.append(float(rng.uniform(-1, 1)))
        if i % 5 == 0:  # a duplicate and an explicit zero
            rows.append(i), cols.append(cols[-1]), vals.append(0.25)
            rows.append(i), cols.append((i + 1) % n), vals.append(0.0)
    rows, cols, vals = np.array(rows), np.array(cols), np.array(vals)
    perm = rng.permutation(rows.size)  # unsorted within rows
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    order = np.argsort(rows, kind="stable")
    rows, cols, vals = rows[order], cols[order], vals[order]
    offsum = np.zeros(n)
    np.add.at(offsum, rows[rows != cols], np.abs(vals[rows != cols]))
    vals[rows == cols] = 1.2 * offsum[rows[rows == cols]] + 1.0
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    c = W.CSR(n, np.cumsum(rp), cols.astype(np.int32), vals)
    # the default pattern is the canonical (duplicate-summed) structure of C, explicit zeros included
    canon = c.to_scipy().tocoo()
    key = np.unique(canon.row.astype(np.int64) * n + canon.col)
    pat = ((key // n).astype(np.int32), (key % n).astype(np.int32))
    compare_run(mc, orc, c, pattern=pat, seed=19, chains=96, burn_in=3, cycles=4, outputs=("diag", "pattern"),
                group_size=16, chain_begin=64)


def test_v5_bit_counters_large_n(mc, orc):
    """n above the byte-counter limit (160k rows): v5 keeps one completion bit
    per row (parity with the sweep barrier); states of sampled chains and the
    diag estimate vs the oracle."""
    c = W.pedigree(170000, seed=91)
    inv = mc.Inverter(c)
    inv.run(23, 64, 1, 2, ("diag",), group_size=32)
    assert inv.kernel_info()["version"] == 5
    r = orc.Matrix(c).run(23, 2, 1, 2, ("diag",), chain_begin=62)
    zg, wg = inv.get_state(62, 2)
    states_match(zg, wg, r["z"], r["w"])
    inv.close()


@pytest.mark.parametrize("kernel", ["v4", "v5", "v6"])
def test_dataflow_long_dependency_chain(mc, orc, monkeypatch, kernel):
    """Worst case for the dataflow kernels: a non-symmetric tridiagonal C
    (every row depends on the previous one, a dependency chain of depth n in
    each sweep) plus a few long-range couplings, with many warps and many
    sweeps in one launch; states and diag / pattern estimates vs the oracle."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    n = 300
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = 3.0
        if i > 0:
            a[i, i - 1] = -0.9
        if i + 1 < n:
            a[i, i + 1] = -0.7
        if i % 37 == 5 and i + 150 < n:
            a[i, i + 150] = 0.4
            a[i + 150, i] = -0.3
    c = W.CSR.from_dense(a)
    for C, th in ((8, "1024"), (32, "1024"), (1 if kernel != "v6" else 2, "256")):
        monkeypatch.setenv("MCINV_C", str(C))
        monkeypatch.setenv("MCINV_THREADS", th)
        compare_run(mc, orc, c, seed=12, chains=64, burn_in=7, cycles=13, outputs=("diag", "pattern"),
                    group_size=8)


@pytest.mark.parametrize("wn,m3", [("32", "0"), ("16", "0"), ("32", "1")])
def test_contraction_tiles_and_staging(mc, orc, monkeypatch, wn, m3):
    """K3 with both warp tilings (MCINV_CONTRACT_WN), the complex product with
    four real products or in the 3-multiplication form (MCINV_CONTRACT_3M, the
    default), and both staging paths: a group size that 16 divides (one
    snapshot sweep per k-chunk) and one that it does not (per-element k / gs),
    complex and real, ragged n (not a multiple of the 64-wide CTA tile)."""
    monkeypatch.setenv("MCINV_CONTRACT_WN", wn)
    monkeypatch.setenv("MCINV_CONTRACT_3M", m3)
    monkeypatch.setenv("MCINV_CONTRACT_OZAKI", "0")  # the DMMA kernels (the Ozaki path has its own test)
    c = W.lattice(5, 3, 0.15, seed=31)  # n = 125: two ragged tiles per dimension
    for gs in (16, 8):
        compare_run(mc, orc, c, seed=9, chains=64, burn_in=2, cycles=5, outputs=("full",), group_size=gs,
                    snapshot_sweeps=3)
    compare_run(mc, orc, W.pedigree(90, seed=32), seed=10, chains=48, burn_in=1, cycles=4, outputs=("full",),
                group_size=48 // 3, snapshot_sweeps=2)


@pytest.mark.parametrize("k", [2, 5])
def test_level2_states_after_sweeps_1_2_and_N_plus_1(mc, orc, k):
    """SURVEY c2 level 2 at full n: z, w after sweeps 1, 2 and N+1 of a chain
    subset (global chain indices 0..7 of the config's run, so the same
    trajectories as the full run), GPU (resumed launches) vs the oracle's
    snapshots of one run, within 1e-12 normwise."""
    c, q, run = W.config(k)
    N, s = run.burn_in, 8
    # snap_sweeps are 0-based: the state after sweep s completes (s = 0: one sweep done)
    r = orc.Matrix(c, q=q).run(run.seed, s, N + 1, 0, (), snap_sweeps=(0, 1, N))
    inv = mc.Inverter(c, q=q)
    done = 0
    for idx, upto in enumerate((1, 2, N + 1)):
        inv.run(run.seed, s, upto - done, 0, (), group_size=1, sweep_begin=done, resume=done > 0)
        done = upto
        zg, wg = inv.get_state(0, s)
        states_match(zg, wg, r["z_snap"][idx], r["w_snap"][idx])
    inv.close()


@pytest.mark.slow
def test_config2_level3_chain_subset(mc, orc):
    """SURVEY c2 level 3 at full n and full sweeps: 16 chains of config 2 (global
    indices 0..15, the same trajectories as in the bench run), 200 + 2000 sweeps,
    diag and pattern estimates vs the oracle within 1e-10 (normwise and
    relative Frobenius)."""
    c, _, run = W.config(2)
    s = 16
    res = compare_run(mc, orc, c, seed=run.seed, chains=s, burn_in=run.burn_in, cycles=run.cycles,
                      outputs=("diag", "pattern"), group_size=8)
    assert np.all(np.isfinite(res["diag"][0]))


@pytest.mark.parametrize("cplx", [True, False])
def test_contraction_ozaki_tcgen05(mc, orc, monkeypatch, cplx):
    """K3 by the Ozaki scheme on the tcgen05 INT8 tensor cores (MCINV_CONTRACT_OZAKI=1:
    exact int8 digit products accumulated in TMEM, fp64 recombination): full C^-1
    estimates and states vs the oracle within the fp64 tolerances, ragged tiles (n not a
    multiple of 128/64), several chunks (ragged last), group sizes 16 and 32."""
    monkeypatch.setenv("MCINV_CONTRACT_OZAKI", "1")
    if cplx:
        c = W.lattice(5, 3, 0.15, seed=31)  # n = 125
        compare_run(mc, orc, c, seed=9, chains=64, burn_in=2, cycles=5, outputs=("full", "diag"), group_size=16,
                    snapshot_sweeps=3)
        compare_run(mc, orc, W.lattice(12, 2, 0.2, seed=33), seed=10, chains=64, burn_in=2, cycles=4, outputs=("full",),
                    group_size=32, snapshot_sweeps=2)
    else:
        compare_run(mc, orc, W.pedigree(150, seed=32), seed=11, chains=64, burn_in=1, cycles=6, outputs=("full",),
                    group_size=16, snapshot_sweeps=4)


@pytest.mark.parametrize("ozaki", ["1", "0"])
@pytest.mark.parametrize("cplx", [True, False])
def test_contraction_wide_row_scales(mc, orc, monkeypatch, cplx, ozaki):
    """Reading R26's bound is relative to each row's and column's own scale (2^e_i, 2^f_j):
    C' = S C S with S = diag(10^U(-4, 4)) spreads the rows of X and Y -- and the entries
    of C'^-1 = S^-1 C^-1 S^-1 -- over 16 orders of magnitude (Gauss-Seidel is invariant
    under the scaling: its iteration matrix is similar to C's). The unscaled estimate
    S est S must match the oracle's within 1e-10, i.e. every element to 1e-10 of its own
    row/column scale, for the Ozaki kernel and for the DMMA kernel."""
    monkeypatch.setenv("MCINV_CONTRACT_OZAKI", ozaki)
    base = W.lattice(5, 3, 0.15, seed=31) if cplx else W.pedigree(150, seed=32)
    s = 10.0 ** np.random.default_rng(77).uniform(-4.0, 4.0, base.n)
    rows = np.repeat(np.arange(base.n), np.diff(base.row_ptr))
    c = W.CSR(base.n, base.row_ptr, base.col, base.val * s[rows] * s[base.col])
    seed, chains, burn, cycles, gs = 12, 64, 2, 5, 16
    inv = mc.Inverter(c)
    inv.run(seed, chains, burn, cycles, ("full",), group_size=gs, snapshot_sweeps=3)
    eg, _ = inv.result("full")
    inv.close()
    r = orc.Matrix(c).run(seed, chains, burn, cycles, ("full",))
    eo, _ = orc.estimate(r["full"], cycles, group_size=gs)
    assert np.max(np.abs(eo)) / np.min(np.abs(np.diag(eo))) > 1e10  # the spread is real
    u = s[:, None] * s[None, :]
    est_match(u * eg, u * eo, what="unscaled full")
