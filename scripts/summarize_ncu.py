"""Distils ncu reports in gpurun_out/ into the committed summaries under
profiles/ (per-kernel key metrics + the launch list share table).

  python scripts/summarize_ncu.py <round-tag>
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "sm__cycles_elapsed.avg",
]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in hdr:
                d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        out.append(d)
    return out


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0][:80]
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
        per[name][0] += 1
        per[name][1] += v * scale
    tot = sum(v[1] for v in per.values()) or 1.0
    return [{"kernel": k, "launches": n, "total_us": round(t, 1), "share": round(t / tot, 4)}
            for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1])]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    summary = {}
    for name in sorted(os.listdir(OUT)):
        if name.endswith(".ncu-rep"):
            summary[name[:-8]] = raw(os.path.join(OUT, name))
    lp = os.path.join(OUT, "launches_bench.csv")
    if os.path.exists(lp):
        summary["launch_list_bench"] = launch_shares(lp)
    with open(os.path.join(PROF, f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:6000])


if __name__ == "__main__":
    main()
