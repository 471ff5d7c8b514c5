"""Chain-parallel oracle runs for the full-size parity tests (test code only).

The oracle (oracle/oracle.c) is single-threaded; chains are independent, so
the runs of a chain subset are spread over host processes, one chain each,
and stacked in chain order. Each worker regenerates the config's matrix from
its seed (workloads/) instead of receiving it by pickle.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np


def _one(args):
    import oracle
    import workloads as W
    k, pure, chain, burn, cycles, outputs, seed, snaps = args
    c, q, _ = W.config(k, pure_gauge=pure)
    pat = None
    if "pattern" in outputs:
        pat = (np.repeat(np.arange(c.n), np.diff(c.row_ptr)).astype(np.int32), c.col)
    m = oracle.Matrix(c, q=q if "trace" in outputs else None, pattern=pat)
    return m.run(seed, 1, burn, cycles, outputs, chain_begin=chain, snap_sweeps=snaps)


def _one_summed(args):
    """_one, with the per-chain outputs kept and the states dropped (sum_outputs)."""
    r = _one(args)
    return {o: r[o] for o in ("diag", "pattern", "full", "trace") if r[o] is not None}


def oracle_chains(k: int, chains, burn: int, cycles: int, outputs=(), seed: int | None = None, pure: bool = False,
                  snaps=(), procs: int | None = None, sum_outputs: bool = False) -> dict:
    """Oracle run of the global chain indices `chains` of BASELINE config k;
    returns the oracle's dict with the per-chain arrays stacked in that order
    (sum_outputs: only the outputs, summed over the chains, shape (1, ...))."""
    import workloads as W
    seed = W.CONFIGS[k]["run"].seed if seed is None else seed
    chains = list(chains)
    procs = procs or min(len(chains), os.cpu_count() or 1)
    jobs = [(k, pure, ch, burn, cycles, tuple(outputs), seed, tuple(snaps)) for ch in chains]
    with mp.get_context("fork").Pool(procs) as pool:
        if sum_outputs:
            acc = {}
            for r in pool.imap(_one_summed, jobs):  # chain order: the same sum on every run
                for o, v in r.items():
                    acc[o] = v.copy() if o not in acc else acc[o] + v
            return acc
        res = pool.map(_one, jobs)
    out = {}
    for key in res[0]:
        if res[0][key] is None:
            out[key] = None
        elif key in ("z_snap", "w_snap"):
            out[key] = np.concatenate([r[key] for r in res], axis=1)
        elif key == "trace_series":  # per-sweep sums over the run's chains
            out[key] = np.sum([r[key] for r in res], axis=0)
        else:
            out[key] = np.concatenate([r[key] for r in res], axis=0)
    return out
