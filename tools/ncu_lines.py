"""Summarise an ncu report: top source lines by stall samples and instructions."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur = None
stall, insts, sass = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
ts = ti = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None:
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        i = int(d.get("Instructions Executed") or 0)
    except ValueError:
        continue
    key = (cur, d["Line No"], r[1][:80])
    stall[key] += s
    insts[key] += i
    if len(r) > 3:
        sass[key][r[3].split()[0] if r[3].split() else ""] += i
    ts += s
    ti += i
print(f"samples {ts} warp-instructions {ti}")
for k, v in stall.most_common(top):
    print(f"{v / max(ts, 1) * 100:5.1f}% stall {insts[k] / max(ti, 1) * 100:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
print("--- by instructions")
for k, v in insts.most_common(top):
    print(f"{stall[k] / max(ts, 1) * 100:5.1f}% stall {v / max(ti, 1) * 100:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
