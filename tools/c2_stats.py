"""Config 2 full-size statistics: diag estimates of 60 sampled rows vs exact solves,
r = (est - exact) / SE, for a given kernel (MCINV_KERNEL) -- diagnosis helper."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import workloads as W
    import paper_cs_0412107_b200 as M
    from tests.test_gpu_parity import _exact_columns
    c, _, run = W.config(2)
    seed = int(sys.argv[1], 0) if len(sys.argv) > 1 else run.seed
    inv = M.Inverter(c)
    inv.run(seed, run.chains, run.burn_in, run.cycles, run.outputs, group_size=run.group_size)
    ed, sd = inv.result("diag")
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(c.n, 60, replace=False))
    X = _exact_columns(c, rows)
    ex = X[rows, np.arange(len(rows))]
    r = (ed[rows] - ex) / sd[rows]
    print(os.environ.get("MCINV_KERNEL", "auto"), hex(seed), inv.kernel_info(), "max|r| %.3f" % np.max(np.abs(r)),
          "mean r^2 %.3f" % np.mean(r * r), "worst row", rows[np.argmax(np.abs(r))], "ed[:3]", ed[rows[:3]])


if __name__ == "__main__":
    main()
