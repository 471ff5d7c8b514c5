"""Small runs of every kernel path for compute-sanitizer (one tool per call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads as W
import paper_cs_0412107_b200 as M

runs = []
c = W.pedigree(300, seed=71)
for ker in ("v4", "v3", "v1"):
    os.environ["MCINV_KERNEL"] = ker
    inv = M.Inverter(c)
    inv.run(1, 64, 2, 3, ("diag", "pattern"), group_size=8)
    runs.append((ker, "pedigree", float(np.abs(inv.result("diag")[0]).sum())))
    inv.close()
L = W.lattice(4, 3, 0.15, seed=72)
q = W.random_q(L.n, 73, 3)
for ker in ("v3", "v4"):
    os.environ["MCINV_KERNEL"] = ker
    inv = M.Inverter(L, q=q)
    outs = ("diag", "trace", "full") if ker == "v3" else ("diag", "full")
    inv.run(2, 48, 1, 3, outs, group_size=16, snapshot_sweeps=2)
    runs.append((ker, "lattice", float(np.abs(inv.result("diag")[0]).sum())))
    inv.close()
os.environ.pop("MCINV_KERNEL")
ph = M.philox(np.arange(64, dtype=np.uint32).reshape(16, 4), 5)
g = M.gaussian(np.arange(64, dtype=np.uint32).reshape(16, 4), 5)
torch.cuda.synchronize()
print("sanitize runs ok", runs, int(ph.sum() % 1000), float(g.sum()))
