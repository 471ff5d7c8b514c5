"""CPU checks of bench.py's roofline bookkeeping: the
algorithmic bytes per site-update and the committed ncu summary it reads."""
import json
import os

import numpy as np

import bench
import workloads as W


def test_algorithmic_bytes_per_site_match_survey_d3():
    # B_site = e (|R_i| + |K_i| + 2) averaged over rows: config 2 111.9 B (f64), config 3 160 B
    # (c128, 4 off-diagonal entries per row and column: 16 (4 + 4 + 2))
    c2, _, _ = W.config(2)
    assert abs(bench.algorithmic_bytes_per_chain_sweep(c2) / c2.n - 111.9) < 0.1
    c3, _, _ = W.config(3)
    assert bench.algorithmic_bytes_per_chain_sweep(c3) / c3.n == 16 * (4 + 4 + 2)
    # a diagonal matrix: only the two stores
    d = W.diagonal(np.array([1.0, 2.0, 3.0]))
    assert bench.algorithmic_bytes_per_chain_sweep(d) == 8 * 2 * 3


def test_committed_ncu_summary_is_complete():
    # the bench line's `traffic` and `roofline.issue` come from this file (one ncu --set full
    # capture of the sweep kernel per workload); the bench workload must be in it
    path = os.path.join(bench.ROOT, "profiles", "ncu_summary.json")
    js = json.load(open(path))
    s = js[W.CONFIGS[2]["name"]]
    assert 40 < s["dram_bytes_per_site"] < 200
    assert 5 < s["warp_inst_per_site"] < 100
    assert bench.committed_traffic(W.CONFIGS[2]["name"]) == s["dram_bytes_per_site"]
    assert bench.committed_summary("no such workload") == {}


def test_config5_bytes_include_the_trace_gathers():
    # config 5 352 B/site = 16 (8 + 8 + 2) + 16 x 4 Q gathers (288 without Q)
    c5, q5, _ = W.config(5)
    assert bench.algorithmic_bytes_per_chain_sweep(c5) / c5.n == 288
    assert bench.algorithmic_bytes_per_chain_sweep(c5, q5) / c5.n == 352


def test_scaling_modes_shard_the_chains():
    """Weak: the config's chains on every rank; strong (default for configs 4
    and 5): BASELINE's total split by whole SE groups, covering it once."""
    for k, total in ((4, 8192), (5, 16384)):
        a = bench.parse(["--config", str(k), "--gpus", "8"])
        assert bench.scaling_mode(a) == "strong"
        _, _, run = W.config(k)
        got = [bench.shard_of(a, run, 8, r) for r in range(8)]
        assert all(t == total for _, _, t in got) and sum(ch for _, ch, _ in got) == total
        assert [cb for cb, _, _ in got] == [r * total // 8 for r in range(8)]
    a = bench.parse(["--gpus", "4"])
    assert bench.scaling_mode(a) == "weak"
    _, _, run = W.config(2)
    assert bench.shard_of(a, run, 4, 3) == (3 * 1024, 1024, 4096)


def test_roofline_bound_is_issue_when_dram_is_below_half_its_peak():
    # round-1 verdict: a kernel whose ncu DRAM bandwidth at the measured rate is below half the
    # peak is not HBM-bound -- the bench labels it by the issue ceiling (the HBM model stays in
    # the object); with enough DRAM traffic it is labelled HBM-bound
    c2, _, r2 = W.config(2)
    name = W.CONFIGS[2]["name"]
    sweeps = r2.burn_in + r2.cycles

    def roof(ms):
        st = {"sweep_ms": ms, "sweep_launches": 1}
        return bench.sweep_roofline(name, c2, None, r2.outputs, r2.chains, sweeps, st, {"version": 6},
                                    {"blocks": 128}, {"sm_mhz": 1965.0}, 148)

    slow = roof(1500.0)  # ~3.0e10 site-updates/s: DRAM ~40% of the peak
    assert slow["dram_frac_of_peak"] < 0.5
    assert slow["bound"] == "issue" and slow["frac"] == slow["issue"]["frac"]
    assert "latency-bound" in slow["note"] and 0 < slow["hbm_model"]["frac"] < 1
    fast = roof(500.0)  # three times the rate: DRAM above half the peak, HBM model above the issue
    assert fast["dram_frac_of_peak"] > 0.5
    assert fast["bound"] == ("issue" if fast["issue"]["frac"] > fast["hbm_model"]["frac"] else "hbm")
