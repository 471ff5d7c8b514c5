"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by CUDA source line:
share of executed warp instructions and of stall samples (profiling helper)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
out, cur, hdr = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] in ("", "Function Name") or hdr is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ie = int(d.get("Instructions Executed", "0"))
        st = int(d.get("Warp Stall Sampling (All Samples)", "0"))
    except ValueError:
        continue
    out.append((cur, r[0], ie, st, r[1][:100]))
tot = sum(o[2] for o in out) or 1
ts = sum(o[3] for o in out) or 1
print(f"total warp instructions {tot}, stall samples {ts}")
for o in sorted(out, key=lambda x: -x[2])[:top]:
    print(f"{o[0]:20s}:{o[1]:>4s} {o[2] / tot * 100:5.1f}% inst {o[3] / ts * 100:5.1f}% stall | {o[4]}")
