"""Summarise gpurun_out ncu captures into profiles/ (committed evidence).

    python tools/summarize_ncu.py <tag> [--full gpurun_out/prof_sweep3.ncu-rep --sites N --workload NAME]
                                        [--launches gpurun_out/launches.csv]
Writes profiles/<tag>_ncu_full.txt (key metrics + stall reasons), profiles/<tag>_launches.txt
(per-kernel launch shares) and updates profiles/ncu_summary.json (DRAM bytes per site-update).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__sass_inst_executed_op_global_red.sum", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    """Metrics of a capture: an .ncu-rep (read with ncu -i) or its `--page raw --csv` export."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--full")
    ap.add_argument("--sites", type=float)
    ap.add_argument("--workload")
    ap.add_argument("--launches")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if a.full:
        recs, units = raw(a.full)
        d = recs[0]
        lines = [f"ncu --set full capture: {a.full} (kernel {d.get('Kernel Name', '')[:90]})"]
        for k in KEYS:
            if k in d:
                lines.append(f"{k:60s} {d[k]:>20s} {units.get(k, '')}")
        st = {k: num(v) for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
        tot = sum(v for v in st.values() if v)
        lines.append("warp stall reasons (share of samples):")
        for k, v in sorted(st.items(), key=lambda t: -(t[1] or 0))[:10]:
            lines.append(f"  {100 * (v or 0) / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
        scale = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        dram = sum((num(d.get(k)) or 0) * scale.get(units.get(k), 1.0)
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        if a.sites:
            lines.append(f"sites (chains x rows x sweeps) in the capture: {a.sites:.6g}")
            lines.append(f"DRAM bytes per site-update: {dram / a.sites:.2f}")
            inst = num(d.get("smsp__inst_executed.sum"))
            if inst:
                lines.append(f"warp instructions per site-update: {inst / a.sites:.2f} (x32 = {32 * inst / a.sites:.0f} "
                             "thread-instruction slots)")
            path = os.path.join(prof, "ncu_summary.json")
            try:
                js = json.load(open(path))
            except (OSError, ValueError):
                js = {}
            js[a.workload] = {"dram_bytes_per_site": dram / a.sites, "capture": os.path.basename(a.full),
                              "tag": a.tag, "sites": a.sites,
                              "warp_inst_per_site": (inst / a.sites) if inst else None,
                              "issue_active_pct": num(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active")),
                              "duration_ms": num(d.get("gpu__time_duration.sum"))}
            json.dump(js, open(path, "w"), indent=1)
        open(os.path.join(prof, f"{a.tag}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))
    if a.launches:
        txt = open(a.launches).read()
        start = txt.find('"ID"')
        rows = list(csv.DictReader(io.StringIO(txt[start:])))
        agg = collections.defaultdict(lambda: [0, 0.0])
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0][:60]
            v = num(r["Metric Value"]) or 0.0
            scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(r.get("Metric Unit"), 1e-9)
            agg[name][0] += 1
            agg[name][1] += v * scale
        tot = sum(v[1] for v in agg.values())
        lines = [f"ncu launch list ({a.launches}): kernel, launches, total s, share of device time"]
        for k, (n, t) in sorted(agg.items(), key=lambda t: -t[1][1]):
            lines.append(f"{k:62s} {n:6d} {t:12.6f} {100 * t / tot:6.2f}%")
        open(os.path.join(prof, f"{a.tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))


if __name__ == "__main__":
    main()
