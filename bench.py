#!/usr/bin/env python
"""Benchmark: Gibbs site-updates/s of the CC inverter on B200 (BASELINE.json metric).

A "step" is one whole run of BASELINE.json configs[1] (config 2: pedigree-like
real non-symmetric C, n = 20,000, 1024 chains per GPU, 200 burn-in + 2000
sampling sweeps, outputs diag + pattern): every sweep of every chain, the
fused accumulation, the moments, the all-reduce across GPUs and the on-device
finalize. value = chains * n * sweeps (all ranks) / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl ours|reference]

N > 1 runs under torchrun (one process per GPU, NCCL); chains are sharded by
global index (weak scaling: 1024 chains per GPU). Timing: CUDA events on the
launch stream, barrier + synchronize on both sides, max over ranks. The state
(n x chains x 16 B = 328 MB) exceeds the 126 MB L2, so no flush is needed.

``--impl reference`` times the oracle (oracle/, single-threaded C, one
process per host core) on a bounded sample of the same workload: the CPU
baseline, not the target.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gibbs site-updates/s (chains·rows/s) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "site-updates/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=2, help="BASELINE.json config number (1-5)")
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0, help="target wall time of one oracle sample")
    p.add_argument("--chains", type=int, default=0, help="override chains per GPU (diagnostics only)")
    return p.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ----------------------------------------------------------------- clocks

class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------- oracle (CPU baseline)

def _oracle_worker(args):
    cfgk, chain0, chains, burn, cyc, seed = args
    import oracle
    import workloads as W
    c, q, run = W.config(cfgk)
    pat = None
    if "pattern" in run.outputs:
        import numpy as np
        pat = (np.repeat(np.arange(c.n), np.diff(c.row_ptr)).astype(np.int32), c.col)
    m = oracle.Matrix(c, q=q, pattern=pat)
    outs = tuple(o for o in run.outputs if o != "full") if c.n > 256 else run.outputs
    t = time.perf_counter()
    m.run(seed, chains, burn, cyc, outs, chain_begin=chain0)
    dt = time.perf_counter() - t
    return chains * c.n * (burn + cyc), dt


def oracle_sample(cfgk: int, target_s: float):
    """Time the oracle, as it stands, on all host cores: one process per core,
    disjoint chains, full n, sweeps sized to ~target_s; burn-in fraction as in
    the config. Returns (rate, cores, sample description)."""
    import oracle
    import workloads as W
    oracle.build()
    c, _, run = W.config(cfgk)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    pilot_s, _ = _oracle_worker((cfgk, 0, 1, 0, 2, run.seed))
    _, pilot_t = _oracle_worker((cfgk, 0, 1, 0, 2, run.seed))
    per_sweep = max(pilot_t / 2, 1e-6)
    sweeps = int(max(2, min(run.burn_in + run.cycles, target_s / per_sweep)))
    burn = max(0, round(sweeps * run.burn_in / (run.burn_in + run.cycles)))
    cyc = max(1, sweeps - burn)
    jobs = [(cfgk, k, 1, burn, cyc, run.seed) for k in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_worker, jobs)
    sites = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    model = "?"
    try:
        with open("/proc/cpuinfo") as f:
            model = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    desc = (f"{W.CONFIGS[cfgk]['name']}: {cores} processes x 1 chain x {burn}+{cyc} sweeps at full n={c.n} "
            f"({sites:.3g} site-updates, outputs {','.join(run.outputs)} minus full when n>256) on {model}; "
            f"single process {pilot_s / pilot_t:.3g} site-updates/s")
    return sites / wall, cores, desc


# ----------------------------------------------------------------- roofline helpers

def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_fp64_peak():
    """FP64 tensor-core yardstick measured on this pool's B200 (tools/fp64_peak.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["zgemm_4096x1024_conjT_tflops"]), "measured cuBLAS ZGEMM (profiles/fp64_peak.json)"
    except (OSError, KeyError, ValueError):
        return 35.0, "fallback (cuBLAS DGEMM measured in round 1)"


def algorithmic_bytes_per_chain_sweep(c) -> int:
    """per site-update, the z gathers of row i (nnz of R_i),
    the w gathers of column i (nnz of K_i) and the two stores, e bytes each:
    sum_i e (|R_i| + |K_i| + 2) = e (2 nnz_offdiag + 2 n) per chain per sweep."""
    import numpy as np
    e = 16 if np.iscomplexobj(c.val) else 8
    rows = np.repeat(np.arange(c.n), np.diff(c.row_ptr))
    off = int(np.sum(rows != c.col))
    return e * (2 * off + 2 * c.n)


def committed_summary(workload: str) -> dict:
    """The committed `ncu --set full` summary of the sweep kernel on this workload
    (profiles/ncu_summary.json; captured on a shorter launch of the same shape, so
    it is stored per site-update): DRAM bytes and warp instructions per site."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload, {})
    except (OSError, ValueError):
        return {}


def committed_traffic(workload: str):
    """DRAM bytes (read + write) per site-update of the sweep kernel (ncu)."""
    return committed_summary(workload).get("dram_bytes_per_site")


# ----------------------------------------------------------------- arms

def reference_arm(args):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    import workloads as W
    vals = []
    cores, desc = None, None
    for s in range(args.warmup + args.steps):
        rate, cores, desc = oracle_sample(args.config, args.cpu_seconds)
        if s >= args.warmup:
            vals.append(rate)
    value = statistics.mean(vals)
    c, _, run = W.config(args.config)
    # the oracle times a bounded sample; the whole step's time at that rate (extrapolated)
    step_sites = run.chains * c.n * (run.burn_in + run.cycles)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_sites / value * 1e3,
            "ms_per_step_kind": "extrapolated from the timed sample", "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": W.CONFIGS[args.config]["dtype"], "data": "synthetic",
            "config": {"workload": W.CONFIGS[args.config]["name"], "n": c.n, "nnz": c.nnz,
                       "chains_per_gpu": run.chains, "burn_in": run.burn_in, "cycles": run.cycles,
                       "outputs": list(run.outputs), "group_size": run.group_size,
                       "matrix_sha256": c.sha256()[:16]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def ours_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import workloads as W
    import paper_cs_0412107_b200 as M
    from paper_cs_0412107_b200.dist import allreduce_moments

    rank, local, world = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    c, q, run = W.config(args.config)
    name = W.CONFIGS[args.config]["name"]
    chains = args.chains or run.chains
    cb = rank * chains
    total_chains = world * chains
    outputs = run.outputs
    sweeps = run.burn_in + run.cycles
    inv = M.Inverter(c, device=local, q=q)

    def barrier():
        if world > 1:
            dist.barrier()

    def step(h: "M.Inverter"):
        h.run(run.seed, chains, run.burn_in, run.cycles, outputs, chain_begin=cb, group_size=run.group_size)
        allreduce_moments(h.accumulators())
        return [h.result(o, total_chains=total_chains, on_device=True) for o in outputs]

    for _ in range(args.warmup):
        step(inv)
    torch.cuda.synchronize()
    barrier()
    inv.stats()  # reset counters
    inv.set_timing(True)
    stream = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks = Clocks(local)
    torch.cuda.synchronize()
    barrier()
    t0.record(stream)
    for _ in range(args.steps):
        step(inv)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    st = inv.stats()
    inv.set_timing(False)
    kinfo = inv.kernel_info()
    if world > 1:
        x = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    sites = total_chains * c.n * sweeps
    value = sites / (ms / 1e3)

    # dominant kernel: the sweep kernel (K1); one launch per step for diag/pattern/trace
    b_chain_sweep = algorithmic_bytes_per_chain_sweep(c)
    sweep_launch_ms = st["sweep_ms"] / max(st["sweep_launches"], 1)
    sweeps_per_launch = sweeps if "full" not in outputs else None
    peak, peak_src = load_peaks()
    roof = None
    if sweeps_per_launch:
        bytes_launch = b_chain_sweep * chains * sweeps_per_launch
        achieved = bytes_launch / (sweep_launch_ms / 1e3) / 1e9
        tps = committed_traffic(name)
        tr = tps * chains * c.n * sweeps_per_launch if tps else None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": tr, "traffic_bytes_per_site": tps,
                "kernel": {3: "sweep3_kernel (v3, level barriers)", 4: "sweep4_kernel (v4, dataflow)",
                           5: "sweep5_kernel (v5, dataflow + TMA-staged plan blocks)",
                           1: "sweep_kernel (v1)"}.get(kinfo["version"], str(kinfo)),
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bytes_launch,
                "algorithmic_bytes_per_site": b_chain_sweep / c.n,
                "sweep_ms_per_launch": sweep_launch_ms,
                "sweep_share_of_step": st["sweep_ms"] / (ms * args.steps)}
        # second ceiling: instruction issue. ncu's warp instructions per
        # site-update on this workload x the SMs holding a CTA x 4 issue slots per clock at the
        # clock measured during the timed region
        ipc = committed_summary(name).get("warp_inst_per_site")
        if ipc and clk.get("sm_mhz"):
            props = torch.cuda.get_device_properties(local)
            sms = min(props.multi_processor_count, -(-chains // max(1, kinfo["chains_per_warp"])))
            ceiling = sms * 4 * clk["sm_mhz"] * 1e6 / ipc
            rate = chains * c.n * sweeps_per_launch / (sweep_launch_ms / 1e3)
            roof["issue"] = {"warp_inst_per_site": ipc, "sms_used": sms, "ceiling": ceiling, "unit": UNIT,
                             "frac": rate / ceiling}

    if "full" in outputs and st["contract_launches"]:
        # the full-inverse contraction dominates (config 3): FP64 tensor-core (DMMA) bound;
        # peak = cuBLAS ZGEMM measured on this box (profiles/fp64_peak.json), else cuBLAS DGEMM
        flops = (8.0 if np.iscomplexobj(c.val) else 2.0) * c.n * c.n * chains * run.cycles
        cms = st["contract_ms"] / args.steps
        fp = load_fp64_peak()
        achieved_tf = flops / (cms / 1e3) / 1e12
        cplx = bool(np.iscomplexobj(c.val))
        m3 = cplx and os.environ.get("MCINV_CONTRACT_3M", "1") != "0"
        roof = {"bound": "tensor", "achieved": achieved_tf, "peak": fp[0], "unit": "TFLOP/s",
                "frac": achieved_tf / fp[0] if fp[0] else None, "traffic": None, "peak_source": fp[1],
                "kernel": "contract_kernel (K3, DMMA mma.sync.m8n8k4.f64" + (", 3-multiplication complex form)"
                                                                             if m3 else ")"),
                "executed_flops_per_step": flops * (0.75 if m3 else 1.0),
                "note": ("achieved counts the algorithmic 8 flops per complex MAC; the 3-multiplication form "
                         "executes 6, so achieved can exceed the ZGEMM peak" if m3 else None),
                "contract_ms_per_step": cms,
                "contract_share_of_step": st["contract_ms"] / (ms * args.steps),
                "algorithmic_flops_per_step": flops}

    # e2e: the public API from host CSR to host estimates, every step
    e2e = None
    if not args.no_e2e:
        h2d = c.row_ptr.nbytes + c.col.nbytes + c.val.nbytes + (q.row_ptr.nbytes + q.col.nbytes + q.val.nbytes
                                                                   if q is not None else 0)
        times = []
        d2h = 0
        for s in range(args.steps + 1):
            torch.cuda.synchronize()
            barrier()
            t = time.perf_counter()
            h = M.Inverter(c, device=local, q=q)
            h.run(run.seed, chains, run.burn_in, run.cycles, outputs, chain_begin=cb, group_size=run.group_size)
            allreduce_moments(h.accumulators())
            res = [h.result(o, total_chains=total_chains) for o in outputs]
            h.close()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            d2h = sum(e.nbytes + s_.nbytes for e, s_ in res)
            if s > 0:  # first iteration is warm-up
                times.append(dt)
        e2e_s = max(times) if times else float("nan")
        if world > 1:
            x = torch.tensor([statistics.mean(times)], device="cuda", dtype=torch.float64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            e2e_s = float(x.item())
        else:
            e2e_s = statistics.mean(times)
        e2e = {"value": sites / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_s * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, desc = oracle_sample(args.config, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": W.CONFIGS[args.config]["dtype"], "data": "synthetic",
                "config": {"workload": name, "n": c.n, "nnz": c.nnz, "chains_per_gpu": chains,
                           "total_chains": total_chains, "burn_in": run.burn_in, "cycles": run.cycles,
                           "outputs": list(outputs), "group_size": run.group_size,
                           "l2": f"inputs larger than L2 (state {c.n * chains * (32 if np.iscomplexobj(c.val) else 16) / 1e6:.0f} MB > 126 MB)",
                           "matrix_sha256": c.sha256()[:16], "kernel": kinfo},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": st["launches"], "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())
