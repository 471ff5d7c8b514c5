"""Full-size parity of the production launch layouts.

The sweep kernel and its launch layout (kernel version, chains per CTA C,
chains per thread K, threads, L2 blocking) depend on n, the chain count and
the outputs -- not on the number of sweeps -- so a short run with BASELINE's
full chain count exercises exactly the layout bench.py times. Those runs are
compared BITWISE-level (state within 1e-12 normwise, Eq. 4/5)
on sampled chains and, for the fused accumulation (Eq. 1/C and Eq. tr,
P:173-182), on whole SE groups' accumulator sums (within 1e-10). The level-3
subsets then run the configs' FULL sweep counts on a few chains (global
indices 0..s-1: the same trajectories as in the full run) and compare the
estimates within 1e-10. Oracle runs are chain-parallel over host processes
(tests/_par.py).
"""
import ctypes

import numpy as np
import pytest

import workloads as W
from tests._par import oracle_chains

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
    a, b = np.asarray(a), np.asarray(b)
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den > 0 else 1.0)


def frob(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def check_states(inv, r, picks, chain0=0):
    for k, ch in enumerate(picks):
        zg, wg = inv.get_state(ch - chain0, 1)
        assert normwise(zg[0], r["z"][k]) < TOL_STATE, (ch, normwise(zg[0], r["z"][k]))
        assert normwise(wg[0], r["w"][k]) < TOL_STATE, (ch, normwise(wg[0], r["w"][k]))


def check_groups(inv, output, groups, r, gs):
    """GPU accumulator sums of whole SE groups vs the oracle's per-chain sums
    of the same chains (r holds them stacked group after group)."""
    got = inv.group_sums(output)
    for k, g in enumerate(groups):
        want = r[output][k * gs:(k + 1) * gs].sum(axis=0)
        assert normwise(got[g], want) < TOL_EST, (output, g, normwise(got[g], want))
        assert frob(got[g], want) < TOL_EST, (output, g, frob(got[g], want))


# ------------------------------------------------------------- production layouts, full chain counts

def test_config4_production_layout(mc):
    """Config 4 (n = 1e6 pedigree, 8192 chains: the level kernel with C = 64
    chains per CTA, 2 chains per thread, 1024 threads) for 2 burn-in + 1
    sampling sweep: chains 0, 4095, 8191 vs the oracle, and the diag sums of
    SE groups 0 and 255 (64 chains) vs the oracle's."""
    c, _, run = W.config(4)
    inv = mc.Inverter(c)
    inv.run(run.seed, run.chains, 2, 1, run.outputs, group_size=run.group_size)
    info = inv.kernel_info()
    lc = inv.launch_config()
    assert info["version"] == 3 and info["chains_per_warp"] == 64 and lc["chains_per_thread"] == 2, (info, lc)
    picks = [0, 4095, 8191]
    r = oracle_chains(4, picks, 2, 1)
    check_states(inv, r, picks)
    chains = list(range(32)) + list(range(8192 - 32, 8192))
    rg = oracle_chains(4, chains, 2, 1, ("diag",))
    check_groups(inv, "diag", [0, 255], rg, 32)
    inv.close()


def test_config5_production_layout(mc):
    """Config 5 (16^4 complex lattice, 16384 chains, diag + trace: the dataflow
    kernel v5 with its trace phase, L2-blocked waves of C = 16 chains per CTA) for 2 burn-in + 1
    sampling sweep: chains 0, 8191, 16383 vs the oracle, and the diag and
    trace (w^dagger Q z, reading R2) sums of SE groups 0 and 511."""
    c, q, run = W.config(5)
    inv = mc.Inverter(c, q=q)
    inv.run(run.seed, run.chains, 2, 1, run.outputs, group_size=run.group_size)
    info = inv.kernel_info()
    assert info["chains_per_warp"] == 16, info
    picks = [0, 8191, 16383]
    r = oracle_chains(5, picks, 2, 1)
    check_states(inv, r, picks)
    chains = list(range(32)) + list(range(16384 - 32, 16384))
    rg = oracle_chains(5, chains, 2, 1, ("diag", "trace"))
    check_groups(inv, "diag", [0, 511], rg, 32)
    check_groups(inv, "trace", [0, 511], rg, 32)
    inv.close()


def test_config3_production_layout(mc):
    """Config 3 (64^2 complex lattice, 2048 chains, full output through the
    DMMA contraction) for 2 burn-in + 3 sampling sweeps in snapshot chunks of
    2 (a ragged last chunk): chains 0 and 2047 vs the oracle, and the full
    X Y^dagger sums of SE group 63 (all 16.7M elements) vs the oracle's."""
    c, _, run = W.config(3)
    inv = mc.Inverter(c)
    inv.run(run.seed, run.chains, 2, 3, ("full",), group_size=run.group_size, snapshot_sweeps=2)
    picks = [0, 2047]
    r = oracle_chains(3, picks, 2, 3)
    check_states(inv, r, picks)
    rg = oracle_chains(3, range(2048 - 32, 2048), 2, 3, ("full",), sum_outputs=True)
    got = inv.group_sums("full", 63, 1)[0]
    want = rg["full"].ravel()
    assert normwise(got, want) < TOL_EST and frob(got, want) < TOL_EST
    inv.close()


# ------------------------------------------------------------- level 3 at full sweeps

def _level3(mc, k, s, outputs, gs):
    c, q, run = W.config(k)
    inv = mc.Inverter(c, q=q if "trace" in outputs else None)
    inv.run(run.seed, s, run.burn_in, run.cycles, outputs, group_size=gs)
    res = {o: inv.result(o) for o in outputs}
    r = oracle_chains(k, range(s), run.burn_in, run.cycles, outputs)
    check_states(inv, r, list(range(s)))
    import oracle
    for o in outputs:
        eo, _ = oracle.estimate(r[o], run.cycles, group_size=gs)
        eg = res[o][0]
        assert normwise(eg, eo) < TOL_EST, (k, o, normwise(eg, eo))
        assert frob(eg, eo) < TOL_EST, (k, o, frob(eg, eo))
    inv.close()


@pytest.mark.slow
def test_config3_level3_full_sweeps(mc):
    """SURVEY c2 level 3: config 3, 4 chains, 200 + 2000 sweeps, full C^-1."""
    _level3(mc, 3, 4, ("full",), 4)


@pytest.mark.slow
def test_config4_level3_full_sweeps(mc):
    """SURVEY c2 level 3: config 4, 8 chains, 100 + 500 sweeps, diag."""
    _level3(mc, 4, 8, ("diag",), 8)


@pytest.mark.slow
def test_config5_level3_full_sweeps(mc):
    """SURVEY c2 level 3: config 5, 8 chains, 200 + 1000 sweeps, diag + trace."""
    _level3(mc, 5, 8, ("diag", "trace"), 8)


# ------------------------------------------------------------- resume, boundary, divergence

def test_resume_full_and_trace_after_burn_in_only(mc):
    """A burn-in-only run (cycles = 0) continued by a resume with cycles keeps
    the workspace layout (snapshot chunk T of the first run), so FULL + TRACE
    + DIAG estimates equal those of one uninterrupted run."""
    c = W.lattice(4, 3, 0.15, seed=41)
    q = W.random_q(c.n, 42, 3)
    outs = ("full", "trace", "diag")
    a = mc.Inverter(c, q=q)
    a.run(3, 64, 4, 0, outs, group_size=16)
    a.run(3, 64, 0, 7, outs, group_size=16, sweep_begin=4, resume=True)
    b = mc.Inverter(c, q=q)
    b.run(3, 64, 4, 7, outs, group_size=16)
    for o in outs:
        ea, sa = a.result(o)
        eb, sb = b.result(o)
        assert normwise(ea, eb) < 1e-12 and normwise(sa, sb) < 1e-9, o
    a.close()
    b.close()


def test_c_abi_library_owned_workspace_resume_and_run_until(mc):
    """Through the C ABI with workspace = NULL (the library owns it): a run,
    a resume of it, and mcinv_run_until (which resumes internally) succeed and
    agree with the same sweeps run in one call."""
    L = mc.load()
    c = W.pedigree(500, seed=43)
    rp = np.ascontiguousarray(c.row_ptr, np.int64)
    col = np.ascontiguousarray(c.col, np.int32)
    val = np.ascontiguousarray(c.val, np.float64)

    def create():
        h = ctypes.c_void_p()
        assert L.mcinv_create(ctypes.byref(h), 0, 1, c.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data) == 0
        return h

    def args(burn, cyc, sweep_begin=0, resume=0):
        return mc._RunArgs(11, 0, 64, burn, cyc, sweep_begin, 1, 0, 16, resume, 0, None, 0, None)

    def diag(h):
        est = np.zeros(c.n)
        assert L.mcinv_result(h, 1, 64, est.ctypes.data, None, c.n, 0) == 0
        return est

    h = create()
    assert L.mcinv_run(h, ctypes.byref(args(3, 5))) == 0
    assert L.mcinv_run(h, ctypes.byref(args(0, 6, 8, 1))) == 0
    e_resumed = diag(h)
    done, rse = ctypes.c_int64(), ctypes.c_double()
    assert L.mcinv_run_until(h, ctypes.byref(args(3, 0)), 1, 1e-12, 4, 12, ctypes.byref(done), ctypes.byref(rse)) == 0
    assert done.value == 12
    e_until = diag(h)
    L.mcinv_destroy(h)
    one = create()
    assert L.mcinv_run(one, ctypes.byref(args(3, 11))) == 0
    e11 = diag(one)
    assert L.mcinv_run(one, ctypes.byref(args(3, 12))) == 0
    e12 = diag(one)
    L.mcinv_destroy(one)
    assert normwise(e_resumed, e11) < 1e-12
    assert normwise(e_until, e12) < 1e-12


@pytest.mark.parametrize("kernel", ["v1", "v3", "v5"])
def test_divergence_is_checked_after_every_sweep(mc, orc, kernel, monkeypatch):
    """Reading R12 as the oracle applies it: a value above 1e12 after ANY
    sweep fails the run, even when the chains come back below 1e12 by its end
    (zero noise from a start of 1e13 on a contracting C: the excursion lasts
    the first sweeps only). The oracle stops at that sweep; the GPU reports
    E_DIVERGED at result (and mcinv_run_status)."""
    monkeypatch.setenv("MCINV_KERNEL", kernel)
    c = W.pedigree(300, seed=44)
    inv = mc.Inverter(c)
    inv.run(1, 32, 0, 0, ("diag",), group_size=32, noise="zero")
    z0 = np.full((32, c.n), 1e13)
    inv.set_state(z0, z0)
    inv.run(1, 32, 0, 400, ("diag",), group_size=32, noise="zero", resume=True)
    zg, _ = inv.get_state()
    assert np.max(np.abs(zg)) < 1e12  # back below the bound at the end
    with pytest.raises(mc.MCInvError) as e:
        inv.result("diag")
    assert e.value.code == 4
    with pytest.raises(orc.OracleError) as eo:
        orc.Matrix(c).run(1, 1, 0, 400, ("diag",), noise=orc.NOISE_ZERO, z_init=z0[0], w_init=z0[0])
    assert eo.value.code == 4
    inv.close()


def test_result_on_device_is_asynchronous_and_run_status_reports(mc):
    """mcinv_result(on_device=1) only enqueues the finalize kernel; a diverged
    run is then reported by mcinv_run_status (E_DIVERGED)."""
    c = W.CSR.from_dense(np.array([[1.0, 3.0], [3.0, 1.0]]))  # sp(T) = 9
    inv = mc.Inverter(c)
    inv.run(1, 32, 200, 1, ("diag",))
    est, se = inv.result("diag", on_device=True)  # no exception: nothing was synchronized
    with pytest.raises(mc.MCInvError) as e:
        inv.run_status()
    assert e.value.code == 4
    inv.close()


def test_recenter_protocol_on_one_gpu(mc):
    """mcinv_recenter: two shards' moment vectors, S1 summed (the all-reduce),
    each recentred on the global mean, M2 summed: equal to the moments of one
    run of all chains (S1 within 1e-12, M2 within 1e-10)."""
    import torch
    c = W.pedigree(2000, seed=7)
    full = mc.Inverter(c)
    full.run(9, 128, 3, 5, ("diag", "pattern"), group_size=32)
    want = full.accumulators().cpu().numpy().copy()
    shards = [mc.Inverter(c) for _ in range(2)]
    for k, s in enumerate(shards):
        s.run(9, 64, 3, 5, ("diag", "pattern"), chain_begin=64 * k, group_size=32)
    accs = [s.accumulators() for s in shards]
    tot = accs[0] + accs[1]
    for a in accs:
        a.copy_(tot)
    m2 = [s.recenter(128) for s in shards]
    m2sum = (m2[0] + m2[1]).cpu().numpy()
    torch.cuda.synchronize()
    nS1 = m2[0].numel()
    assert normwise(tot.cpu().numpy()[:nS1], want[:nS1]) < 1e-12
    assert normwise(m2sum, want[nS1:2 * nS1]) < 1e-10


def test_config2_production_layout(mc):
    """Config 2 as bench.py times it (1024 chains: the v6 dataflow kernel, C = 8,
    two chains per thread, 512 threads) for 2 burn-in + 1 sampling sweep: chains
    0, 513, 1023 vs the oracle, and the diag and pattern sums of SE groups 0 and
    31 vs the oracle's."""
    c, _, run = W.config(2)
    inv = mc.Inverter(c)
    inv.run(run.seed, run.chains, 2, 1, run.outputs, group_size=run.group_size)
    info, lc = inv.kernel_info(), inv.launch_config()
    assert info["version"] == 6 and lc["chains_per_thread"] == 2, (info, lc)
    picks = [0, 513, 1023]
    r = oracle_chains(2, picks, 2, 1)
    check_states(inv, r, picks)
    chains = list(range(32)) + list(range(1024 - 32, 1024))
    rg = oracle_chains(2, chains, 2, 1, ("diag", "pattern"))
    check_groups(inv, "diag", [0, 31], rg, 32)
    check_groups(inv, "pattern", [0, 31], rg, 32)
    inv.close()
