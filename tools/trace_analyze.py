"""Offline analysis of a sweep6 MCINV_TRACE dump (tools/trace_v6.py): phase durations per warp
item, the sweep time, and how long items wait on their lower neighbours."""
import sys
import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.bin"
    a = np.fromfile(path, dtype=np.int64).reshape(-1, 20)
    g, s, t = a[:, 0], a[:, 1], a[:, 2:9].astype(np.float64)
    rows = a[:, 9:17]
    names = ["plan wait", "prefetch+noise", "dep waits", "gathers+fma+store", "publish", "accumulate"]
    d = np.diff(t, axis=1)
    tot = t[:, 6] - t[:, 0]
    print(f"items {len(a)}; mean item {tot.mean():.0f} cycles")
    for k, nm in enumerate(names):
        print(f"  {nm:20s} mean {d[:, k].mean():7.0f}  median {np.median(d[:, k]):7.0f}  p90 {np.percentile(d[:, k], 90):7.0f}  share {d[:, k].sum() / tot.sum():.3f}")
    for sw in np.unique(s):
        m = s == sw
        print(f"sweep {sw}: span {t[m, 6].max() - t[m, 0].min():.0f} cycles, items {m.sum()}")
    # the item gap: start of an item minus the end of the previous item on the same warp
    import workloads as W
    c, q, run = W.config(2)
    n = c.n
    pub = {}
    for it in range(len(a)):
        for r in rows[it]:
            if r >= 0:
                pub[(int(s[it]), int(r))] = t[it, 4]
    rp, col = c.row_ptr, c.col
    low = [set() for _ in range(n)]
    for i in range(n):
        for j in col[rp[i]:rp[i + 1]]:
            j = int(j)
            if j < i:
                low[i].add(j)
            elif j > i:
                low[j].add(i)
    late = []
    for it in range(len(a)):
        last = 0.0
        for r in rows[it]:
            if r < 0:
                continue
            for j in low[int(r)]:
                pt = pub.get((int(s[it]), j))
                if pt is not None:
                    last = max(last, pt)
        late.append(last - t[it, 2])  # > 0: a lower neighbour published after the waits began
    late = np.array(late)
    print(f"dependency published after the item reached its waits: {np.mean(late > 0):.3f} of items; "
          f"mean lateness of those {late[late > 0].mean():.0f} cycles")
    # sweep start/end profile: how many items are in flight over time in sweep 1
    sw = np.unique(s)[0]
    m = s == sw
    t0 = t[m, 0].min()
    span = t[m, 6].max() - t0
    bins = np.linspace(0, span, 21)
    st = t[m, 0] - t0
    hist = np.histogram(st, bins)[0]
    print("item starts per 5% of the sweep:", hist.tolist())
    # the barrier wait: per warp, the last item's end vs the sweep end
    ends = []
    for w in range(16):
        mw = m & (g % 16 == w)
        ends.append(t[mw, 6].max() - t0)
    print("per-warp last item end (fraction of sweep):", np.round(np.array(ends) / span, 3).tolist())


if __name__ == "__main__":
    main()
