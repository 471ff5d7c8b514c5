#!/usr/bin/env python
"""Benchmark: Gibbs site-updates/s of the CC inverter on B200 (BASELINE.json metric).

A "step" is one whole run of a BASELINE.json config through the C ABI: every
sweep of every chain (burn-in included), the fused accumulation, the moments,
the cross-rank reduction of the moments and the on-device finalize.
value = chains * n * sweeps (all ranks) / step time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--scaling auto|weak|strong]
                    [--impl ours|reference] [--no-per-config] [--no-e2e] [--no-cpu-baseline]

Default: config 2 (configs[1]: pedigree-like real C, n = 20,000, 1024 chains
per GPU, 200 + 2000 sweeps, diag + pattern), weak scaling. Configs 4 and 5
default to strong scaling: BASELINE's total chains (8192 / 16384) are split
over the N ranks by whole SE groups (dist.shard). With --gpus N > 1 outside
torchrun, bench.py launches itself under torch.distributed.run with N ranks
(one process per GPU, NCCL). Timing: CUDA events on the launch stream, a
barrier + synchronize on both sides, max over ranks. Every config's state
exceeds the 126 MB L2 (config 2: 328 MB), so no flush is needed.

At N = 1 the line also carries `per_config`: one full step of each of configs
3, 4 and 5 (after the timed loop), with their roofline numbers.

``--impl reference`` times the oracle (oracle/, single-threaded C, one
process per host core) on a bounded sample of the same workload: the CPU
baseline, not the target.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gibbs site-updates/s (chains·rows/s) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "site-updates/s"


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=2, help="BASELINE.json config number (1-5)")
    p.add_argument("--scaling", choices=["auto", "weak", "strong"], default="auto",
                   help="weak: the config's chains per GPU; strong: its total chains split over GPUs "
                        "(auto: strong for configs 4 and 5, weak otherwise)")
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-per-config", action="store_true", help="skip the one-step runs of configs 3, 4, 5")
    p.add_argument("--cpu-seconds", type=float, default=8.0, help="target wall time of one oracle sample")
    p.add_argument("--chains", type=int, default=0, help="override chains per GPU (diagnostics only)")
    return p.parse_args(argv)


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def scaling_mode(args) -> str:
    if args.scaling != "auto":
        return args.scaling
    return "strong" if args.config in (4, 5) else "weak"


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run with
    N ranks on this node (the driver's own launch line), passing stdout through."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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


def _cpu_clocks() -> str:
    """lscpu's model and clock range, for the baseline's description."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
    except (OSError, subprocess.SubprocessError):
        return "lscpu unavailable"
    d = {}
    for line in out.splitlines():
        if ":" in line:
            k, v = line.split(":", 1)
            d[k.strip()] = v.strip()
    mhz = d.get("CPU max MHz")
    if mhz is None:  # VMs often hide the range: the current clock from /proc/cpuinfo
        try:
            with open("/proc/cpuinfo") as f:
                cur = [float(l.split(":", 1)[1]) for l in f if l.startswith("cpu MHz")]
            mhz = f"{max(cur):.0f} (current, /proc/cpuinfo)" if cur else "?"
        except (OSError, ValueError):
            mhz = "?"
    return (f"{d.get('Model name', '?')}, {d.get('CPU(s)', '?')} CPUs, max {mhz} MHz, "
            f"min {d.get('CPU min MHz', '?')} MHz")


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
    desc = (f"{W.CONFIGS[cfgk]['name']}: {cores} processes x 1 chain x {burn}+{cyc} sweeps at full n={c.n} "
            f"({sites:.3g} site-updates, outputs {','.join(run.outputs)} minus full when n>256) on "
            f"{_cpu_clocks()}; single process {pilot_s / pilot_t:.3g} site-updates/s")
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


def algorithmic_bytes_per_chain_sweep(c, q=None) -> int:
    """per site-update, the z gathers of row i (nnz of R_i),
    the w gathers of column i (nnz of K_i) and the two stores, e bytes each:
    sum_i e (|R_i| + |K_i| + 2) = e (2 nnz_offdiag + 2 n) per chain per sweep;
    with the trace output also the z gathers of row i of Q (e nnz(Q): config 5's
    352 B/site = 288 + 4 x 16)."""
    import numpy as np
    e = 16 if np.iscomplexobj(c.val) else 8
    rows = np.repeat(np.arange(c.n), np.diff(c.row_ptr))
    off = int(np.sum(rows != c.col))
    return e * (2 * off + 2 * c.n) + (e * int(q.nnz) if q is not None else 0)


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


KERNELS = {3: "sweep3_kernel (v3, level barriers)", 4: "sweep4_kernel (v4, dataflow)",
           5: "sweep5_kernel (v5, dataflow + TMA-staged plan blocks)",
           6: "sweep6_kernel (v6, dataflow + TMA-staged plan blocks, two chains per thread)",
           1: "sweep_kernel (v1)"}


def sweep_roofline(name, c, q, outputs, chains, sweeps, st, kinfo, lconf, clk, sms_total):
    """Roofline of the sweep kernel K1 over its launches: achieved algorithmic bytes
     per launch / launch time against the measured HBM peak, and the
    instruction-issue ceiling from the committed ncu warp instructions per
    site. `bound` names the nearer of the two ceilings (the larger fraction), or the issue
    ceiling when ncu's DRAM bandwidth at this rate is below half the peak (the kernel is then
    latency-bound, not HBM-bound); both stay in the object, with that DRAM fraction."""
    launch_ms = st["sweep_ms"] / max(st["sweep_launches"], 1)
    per_launch_sweeps = sweeps / max(st["sweep_launches"], 1)
    sites_launch = chains * c.n * per_launch_sweeps
    rate = sites_launch / (launch_ms / 1e3)
    bpc = algorithmic_bytes_per_chain_sweep(c, q if "trace" in outputs else None)
    peak, peak_src = load_peaks()
    bytes_launch = bpc * chains * per_launch_sweeps
    achieved = bytes_launch / (launch_ms / 1e3) / 1e9
    summ = committed_summary(name)
    tps = summ.get("dram_bytes_per_site")
    hbm = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "algorithmic_bytes_per_site": bpc / c.n, "algorithmic_bytes_per_launch": bytes_launch,
           "peak_source": peak_src}
    out = {"kernel": KERNELS.get(kinfo["version"], str(kinfo)), "launch": dict(kinfo, **lconf),
           "sweep_ms_per_launch": launch_ms, "site_updates_per_s": rate,
           "traffic": tps * sites_launch if tps else None, "traffic_bytes_per_site": tps,
           "hbm_model": hbm}
    ipc = summ.get("warp_inst_per_site")
    issue = None
    if ipc and clk.get("sm_mhz"):
        sms = min(sms_total, lconf.get("blocks") or sms_total)
        peak_i = sms * 4 * clk["sm_mhz"] * 1e6  # warp instructions / s: 4 schedulers per SM
        issue = {"achieved": rate * ipc, "peak": peak_i, "unit": "warp-inst/s", "frac": rate * ipc / peak_i,
                 "warp_inst_per_site": ipc, "sms_used": sms, "ceiling_site_updates_per_s": peak_i / ipc,
                 "capture": summ.get("tag")}
        out["issue"] = issue
    dram_frac = (tps * rate / 1e9 / peak) if tps else None
    out["dram_frac_of_peak"] = dram_frac
    if issue is not None and (issue["frac"] > hbm["frac"] or (dram_frac is not None and dram_frac < 0.5)):
        # DRAM below half its peak (ncu): HBM is not what binds the kernel -- it is latency-bound
        # (DESIGN.md §4), and the issue ceiling is the compute-side yardstick (round-1 verdict);
        # the HBM model stays in `hbm_model`
        out.update(bound="issue", achieved=issue["achieved"], peak=issue["peak"], unit="warp-inst/s",
                   frac=issue["frac"])
        if dram_frac is not None and dram_frac < 0.5:
            out["note"] = (f"latency-bound: ncu DRAM at {dram_frac:.0%} of peak at this rate; "
                           f"HBM model {hbm['frac']:.2f}, issue ceiling {issue['frac']:.2f}")
    else:
        out.update(bound="hbm", achieved=achieved, peak=peak, unit="GB/s", frac=achieved / peak)
    return out


def load_int8_peak():
    """Dense int8 tensor peak: the measured bf16 matmul (MEASURED_PEAKS.json) x the guide's
    nominal int8/bf16 ratio (4.5 / 2.25 PFLOP/s)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return 2.0 * float(json.load(f)["bf16_tflops"]), "measured bf16 x 2 (MEASURED_PEAKS.json, nominal int8/bf16)"
    except (OSError, KeyError, ValueError):
        return 4500.0, "fallback (nominal dense int8)"


OZAKI_DIGITS = 6  # contract_ozaki.cu kNS


def contract_roofline(c, chains, cycles, st, steps, group_size=32):
    """K3 (X Y^dagger over snapshot chunks): algorithmic flops 8 n^2 per complex sample
    (2 n^2 real). The default for n >= 256 is the Ozaki scheme on tcgen05 int8 -- bound:
    the int8 tensor pipe, executed int8 ops (NS(NS+1)/2 digit pairs x 2 n^2 K' per pass)
    against the int8 peak; below, the DMMA kernel against cuBLAS ZGEMM."""
    import numpy as np
    cplx = bool(np.iscomplexobj(c.val))
    flops = (8.0 if cplx else 2.0) * c.n * c.n * chains * cycles
    cms = st["contract_ms"] / steps
    achieved_tf = flops / (cms / 1e3) / 1e12
    oz_env = os.environ.get("MCINV_CONTRACT_OZAKI")
    if (c.n >= 256 and oz_env is None) or (oz_env is not None and oz_env != "0"):
        pairs = OZAKI_DIGITS * (OZAKI_DIGITS + 1) // 2
        kp_per_sample = 2 if cplx else 1  # K' = 2K for complex ([re | im]), two passes
        passes = 2 if cplx else 1
        ops = 2.0 * pairs * c.n * c.n * chains * cycles * kp_per_sample * passes
        pk = load_int8_peak()
        achieved = ops / (cms / 1e3) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": pk[0], "unit": "TOP/s (int8)",
                "frac": achieved / pk[0], "traffic": None, "peak_source": pk[1],
                "kernel": f"ozaki_gemm_kernel (K3, Ozaki scheme: {OZAKI_DIGITS} int8 digits, tcgen05.mma kind::i8, "
                          "TMEM accumulators)",
                "fp64_equivalent_tflops": achieved_tf, "executed_int8_ops_per_step": ops,
                "note": "contract_ms includes the digit slicing (about 9% of it); the UMMA microbenchmark "
                        "(tools/micro/umma_bench.cu) sustains 4.76 int8 POP/s at N >= 128",
                "contract_ms_per_step": cms, "algorithmic_flops_per_step": flops,
                "dmma_yardstick_tflops": load_fp64_peak()[0]}
    fp = load_fp64_peak()
    m3 = cplx and os.environ.get("MCINV_CONTRACT_3M", "1") != "0"
    return {"bound": "tensor", "achieved": achieved_tf, "peak": fp[0], "unit": "TFLOP/s",
            "frac": achieved_tf / fp[0] if fp[0] else None, "traffic": None, "peak_source": fp[1],
            "kernel": "contract_kernel (K3, DMMA mma.sync.m8n8k4.f64" + (", 3-multiplication complex form)"
                                                                         if m3 else ")"),
            "executed_flops_per_step": flops * (0.75 if m3 else 1.0),
            "note": ("achieved counts the algorithmic 8 flops per complex MAC; the 3-multiplication form "
                     "executes 6, so achieved can exceed the ZGEMM peak" if m3 else None),
            "contract_ms_per_step": cms, "algorithmic_flops_per_step": flops}


def config_dict(args, c, q, run, world, chains_rank, total_chains, scaling):
    """The workload description, identical in both arms."""
    import numpy as np
    import workloads as W
    return {"workload": W.CONFIGS[args.config]["name"], "n": c.n, "nnz": c.nnz,
            "chains_per_gpu": chains_rank, "total_chains": total_chains, "scaling": scaling,
            "burn_in": run.burn_in, "cycles": run.cycles, "outputs": list(run.outputs),
            "group_size": run.group_size, "noise": "gauss (Philox4x32-10 + Box-Muller)",
            "l2": f"inputs larger than L2 (state {c.n * chains_rank * (32 if np.iscomplexobj(c.val) else 16) / 1e6:.0f}"
                  f" MB per GPU > 126 MB): no flush",
            "matrix_sha256": c.sha256()[:16], "q_nnz": int(q.nnz) if q is not None else 0}


def shard_of(args, run, world, rank):
    """(chain_begin, chains of this rank, total chains) for the scaling mode."""
    from paper_cs_0412107_b200.dist import shard
    mode = scaling_mode(args)
    if mode == "strong":
        total = args.chains * world if args.chains else run.chains
        cb, ch = shard(total, world, rank, run.group_size)
        return cb, ch, total
    ch = args.chains or run.chains
    return rank * ch, ch, world * ch


# ----------------------------------------------------------------- arms

def reference_arm(args):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    import workloads as W
    world = max(world, args.gpus)
    vals = []
    cores, desc = None, None
    for s in range(args.warmup + args.steps):
        rate, cores, desc = oracle_sample(args.config, args.cpu_seconds)
        if s >= args.warmup:
            vals.append(rate)
    value = statistics.mean(vals)
    c, q, run = W.config(args.config)
    _, ch0, total = shard_of(args, run, world, 0)
    step_sites = total * c.n * (run.burn_in + run.cycles)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_sites / value * 1e3,
            "ms_per_step_kind": "extrapolated from the timed sample", "higher_is_better": True,
            "scaling": scaling_mode(args), "vs_baseline": None, "dtype": W.CONFIGS[args.config]["dtype"],
            "data": "synthetic", "config": config_dict(args, c, q, run, world, ch0, total, scaling_mode(args)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def one_config_step(k: int, device: int, sms: int):
    """One full step of BASELINE config k on this GPU (the per_config block): value,
    sweep roofline (and K3 for the full output), clocks."""
    import torch
    import workloads as W
    import paper_cs_0412107_b200 as M
    c, q, run = W.config(k)
    name = W.CONFIGS[k]["name"]
    inv = M.Inverter(c, device=device, q=q)
    # lazily loaded kernel modules and the level plan: a 1-sweep run of the same layout
    inv.run(run.seed, run.chains, 0, 1, run.outputs, group_size=run.group_size)
    torch.cuda.synchronize()
    inv.stats()
    inv.set_timing(True)
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = Clocks(device)
    t0.record(stream)
    inv.run(run.seed, run.chains, run.burn_in, run.cycles, run.outputs, group_size=run.group_size)
    res = [inv.result(o, total_chains=run.chains, on_device=True) for o in run.outputs]
    t1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    inv.run_status()
    ms = t0.elapsed_time(t1)
    st = inv.stats()
    kinfo, lconf = inv.kernel_info(), inv.launch_config()
    sweeps = run.burn_in + run.cycles
    sites = run.chains * c.n * sweeps
    out = {"workload": name, "chains": run.chains, "burn_in": run.burn_in, "cycles": run.cycles,
           "outputs": list(run.outputs), "value": sites / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
           "steps": 1, "clocks": clk, "gpu_launches": st["launches"],
           "sweep": sweep_roofline(name, c, q, run.outputs, run.chains, sweeps, st, kinfo, lconf, clk, sms)}
    if "full" in run.outputs and st["contract_launches"]:
        out["contraction"] = contract_roofline(c, run.chains, run.cycles, st, 1)
        out["contraction"]["contract_share_of_step"] = st["contract_ms"] / ms
    del res
    inv.close()
    del inv
    torch.cuda.empty_cache()
    return out


def ours_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import workloads as W
    import paper_cs_0412107_b200 as M
    from paper_cs_0412107_b200.dist import reduce_moments

    rank, local, world = env_rank()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    c, q, run = W.config(args.config)
    name = W.CONFIGS[args.config]["name"]
    mode = scaling_mode(args)
    cb, chains, total_chains = shard_of(args, run, world, rank)
    outputs = run.outputs
    sweeps = run.burn_in + run.cycles
    inv = M.Inverter(c, device=local, q=q)
    sms = torch.cuda.get_device_properties(local).multi_processor_count

    def barrier():
        if world > 1:
            dist.barrier()

    def step(h: "M.Inverter"):
        h.run(run.seed, chains, run.burn_in, run.cycles, outputs, chain_begin=cb, group_size=run.group_size)
        reduce_moments(h, total_chains)
        return [h.result(o, total_chains=total_chains, on_device=True) for o in outputs]

    for _ in range(args.warmup):
        step(inv)
    torch.cuda.synchronize()
    inv.run_status()
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
    inv.run_status()  # divergence / watchdog of the timed runs
    ms = t0.elapsed_time(t1) / args.steps
    st = inv.stats()
    inv.set_timing(False)
    kinfo, lconf = inv.kernel_info(), inv.launch_config()
    if world > 1:
        x = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    sites = total_chains * c.n * sweeps
    value = sites / (ms / 1e3)

    roof = None
    if "full" not in outputs:
        roof = sweep_roofline(name, c, q, outputs, chains, sweeps * args.steps, st, kinfo, lconf, clk, sms)
        roof["sweep_share_of_step"] = st["sweep_ms"] / (ms * args.steps)
    elif st["contract_launches"]:
        roof = contract_roofline(c, chains, run.cycles, st, args.steps)
        roof["contract_share_of_step"] = st["contract_ms"] / (ms * args.steps)

    # e2e: the public API from host CSR to host estimates, every step (mean over K steps)
    e2e = None
    if not args.no_e2e:
        h2d = c.row_ptr.nbytes + c.col.nbytes + c.val.nbytes + (q.row_ptr.nbytes + q.col.nbytes + q.val.nbytes
                                                                   if q is not None else 0)
        times = []
        d2h = 0
        inv.close()
        del inv
        for s in range(args.steps + 1):
            torch.cuda.synchronize()
            barrier()
            t = time.perf_counter()
            h = M.Inverter(c, device=local, q=q)
            h.run(run.seed, chains, run.burn_in, run.cycles, outputs, chain_begin=cb, group_size=run.group_size)
            reduce_moments(h, total_chains)
            res = [h.result(o, total_chains=total_chains) for o in outputs]
            h.close()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            d2h = sum(e.nbytes + s_.nbytes for e, s_ in res)
            if s > 0:  # first iteration is warm-up
                times.append(dt)
        e2e_s = statistics.mean(times)
        if world > 1:
            x = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            e2e_s = float(x.item())
        e2e = {"value": sites / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_s * 1e3, "statistic": "mean over the timed steps, max over ranks"}
    else:
        inv.close()
        del inv
    torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, desc = oracle_sample(args.config, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}

    per_config = None
    if world == 1 and not args.no_per_config and args.config == 2 and not args.chains:
        per_config = {}
        for k in (3, 4, 5):
            try:
                per_config[W.CONFIGS[k]["name"]] = one_config_step(k, local, sms)
            except Exception as e:  # reported, never silently dropped
                per_config[W.CONFIGS[k]["name"]] = {"error": repr(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": mode,
                "vs_baseline": None, "dtype": W.CONFIGS[args.config]["dtype"], "data": "synthetic",
                "config": config_dict(args, c, q, run, world, chains, total_chains, mode),
                "kernel": dict(kinfo, **lconf),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": st["launches"], "clocks": clk, "per_config": per_config}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.gpus > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init lines (one per rank) stay visible
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return ours_arm(args)


if __name__ == "__main__":
    sys.exit(main())
