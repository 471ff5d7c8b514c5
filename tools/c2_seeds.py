"""Config 2 full-size statistics over several run seeds (diagnosis helper): max|r| and
mean r^2 of 60 sampled diag elements against exact solves, r = (est - exact) / SE."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import workloads as W
    import paper_cs_0412107_b200 as M
    from tests.test_gpu_parity import _exact_columns
    c, _, run = W.config(2)
    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(c.n, 60, replace=False))
    X = _exact_columns(c, rows)
    ex = X[rows, np.arange(len(rows))]
    inv = M.Inverter(c)
    for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
        seed = run.seed + 0x10000 * k
        inv.run(seed, run.chains, run.burn_in, run.cycles, ("diag",), group_size=run.group_size)
        ed, sd = inv.result("diag")
        r = (ed[rows] - ex) / sd[rows]
        print(hex(seed), "max|r| %.3f" % np.max(np.abs(r)), "mean r^2 %.3f" % np.mean(r * r), flush=True)


if __name__ == "__main__":
    main()
