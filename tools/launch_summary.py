"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui, mi = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = {"us": v / 1e3, "ms": v, "ns": v / 1e6, "usecond": v / 1e3, "msecond": v, "nsecond": v / 1e6}.get(r[ui], v)
    agg[re.sub(r"\(.*", "", r[ki])[:80]][0] += 1
    agg[re.sub(r"\(.*", "", r[ki])[:80]][1] += v
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.3f} ms {100 * t / tot:5.1f}% {c:6d}  {k}")
