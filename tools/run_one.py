"""One short CC run of a BASELINE config through the C ABI (for ncu / quick timing).

    python tools/run_one.py --config 2 --sweeps 12 [--chains 1024] [--repeat 1]
Prints per-run device time of the sweep kernel and site-updates/s.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--sweeps", type=int, default=12)
    ap.add_argument("--burn", type=int, default=2)
    ap.add_argument("--chains", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--outputs", default="")
    ap.add_argument("--group-size", type=int, default=0, help="SE group size (default: the config's)")
    ap.add_argument("--noise", default="gauss", choices=["gauss", "z2", "zero"])
    ap.add_argument("--dirac", type=int, default=0, help="free Wilson-Dirac N^4 lattice (trace, Q = I) instead")
    a = ap.parse_args()
    import torch
    import workloads as W
    import paper_cs_0412107_b200 as M
    c, q, run = W.config(a.config)
    if a.dirac:
        c = W.dirac(a.dirac)
        q = W.identity_q(c.n)
        run = W.RunSpec(chains=2048, burn_in=30, cycles=200, outputs=("trace",), seed=0x5EED0012, group_size=32)
    chains = a.chains or run.chains
    outs = tuple(a.outputs.split(",")) if a.outputs else run.outputs
    inv = M.Inverter(c, q=q)
    inv.set_timing(True)
    for _ in range(a.repeat):
        t = time.perf_counter()
        inv.run(run.seed, chains, a.burn, a.sweeps - a.burn, outs, group_size=a.group_size or run.group_size, noise=a.noise)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        st = inv.stats()
        sites = chains * c.n * a.sweeps
        print(f"config {a.config} chains {chains} sweeps {a.sweeps}: wall {dt * 1e3:.1f} ms, sweep kernel "
              f"{st['sweep_ms']:.1f} ms ({st['sweep_launches']} launches), contraction {st['contract_ms']:.1f} ms, "
              f"{sites / (st['sweep_ms'] / 1e3):.3e} "
              f"site-updates/s, kernel {inv.kernel_info()}", flush=True)


if __name__ == "__main__":
    main()
