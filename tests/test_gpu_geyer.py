"""NEXT-2 remainder: Geyer's effective sample size and the paper's stopping rule
(PAPER.md:354-360), GPU (C ABI) vs the oracle on the same seeds.

The GPU keeps, per sampling sweep, the realized trace w^dagger Q z summed over
the run's chains (reading R2), reduced inside the sweep kernel; mcinv_geyer
runs Geyer's initial positive sequence estimator on it. The oracle produces
the same series from its chain-by-chain run (orc_run trace_series) and its own
estimator (orc_geyer, pinned in test_oracle_pins)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0412107_b200 as M
    M.load()
    return M


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("kernel", ["auto", "v1"])
def test_trace_series_and_geyer_match_oracle(mc, orc, kernel, monkeypatch):
    if kernel != "auto":
        monkeypatch.setenv("MCINV_KERNEL", kernel)
    c = W.lattice(4, 2, 0.2, seed=71)
    q = W.random_q(c.n, 72, 3)
    inv = mc.Inverter(c, q=q)
    inv.run(9, 64, 3, 20, ("trace", "diag"), group_size=16, trace_series=60)
    inv.run(9, 64, 0, 40, ("trace", "diag"), group_size=16, sweep_begin=23, resume=True, trace_series=60)
    g = inv.geyer()
    r = orc.Matrix(c, q=q).run(9, 64, 3, 60, ("trace",))
    s = r["trace_series"]
    for comp, part in (("re", s.real), ("im", s.imag)):
        o = orc.geyer(part)
        for key in ("mean", "gamma0", "sigma2", "ess"):
            assert rel(g[comp][key], o[key]) < 1e-10, (comp, key, g[comp][key], o[key])
    est, _ = inv.result("trace")
    assert rel(g["re"]["estimate"], est.real) < 1e-12
    inv.close()


def test_run_until_geyer_paper_rule(mc, orc):
    """Blocks of check_cycles sampling sweeps until the Geyer relative SE of the
    trace is below the tolerance (the paper checks every 100 cycles); the
    estimate and the Geyer SE equal the oracle's for the same total sweeps."""
    c = W.lattice(3, 2, 0.2, seed=73)
    q = W.identity_q(c.n)
    inv = mc.Inverter(c, q=q)
    done, rse = inv.run_until_geyer(19, 32, 10, ("trace",), 2e-3, check_cycles=50, max_cycles=5000, group_size=8)
    assert done % 50 == 0 and rse < 2e-3
    g = inv.geyer()
    est, _ = inv.result("trace")
    r = orc.Matrix(c, q=q).run(19, 32, 10, done, ("trace",))
    eo, _ = orc.estimate(r["trace"], done, group_size=8)
    assert rel(est.real, eo.real) < 1e-10
    o = orc.geyer(r["trace_series"].real)
    se_o = np.sqrt(o["sigma2"] / done) / 32
    assert rel(g["re"]["se"], se_o) < 1e-9
    # the stopping rule: relative Geyer SE (moduli) below the tolerance now, not one block earlier
    assert np.hypot(g["re"]["se"], g["im"]["se"]) / abs(est) < 2e-3
    if done > 50:
        r2 = orc.Matrix(c, q=q).run(19, 32, 10, done - 50, ("trace",))
        s2 = r2["trace_series"]
        o2r, o2i = orc.geyer(s2.real), orc.geyer(s2.imag)
        rse_prev = np.hypot(np.sqrt(o2r["sigma2"] / (done - 50)), np.sqrt(max(o2i["sigma2"], 0) / (done - 50))) / \
            abs(s2.mean())
        assert rse_prev >= 2e-3
    inv.close()
