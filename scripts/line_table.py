"""Per-source-line totals (warp-stall samples, warp instructions executed)
from `ncu -i rep --page source --csv --print-source cuda,sass`.
usage: line_table.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
samp = hdr.index("Warp Stall Sampling (All Samples)")
inst = hdr.index("Instructions Executed")
agg = {}
line, src = None, ""
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0]:
        line, src = r[0], r[1]
    if line is None or not r[2].startswith("0x"):  # SASS rows only (the line rows repeat their totals)
        continue
    num = lambda x: int(x) if x.strip().lstrip('-').isdigit() else 0
    s = num(r[samp])
    n = num(r[inst])
    a = agg.setdefault(line, [0, 0, src])
    a[0] += s
    a[1] += n
S = sum(a[0] for a in agg.values())
N = sum(a[1] for a in agg.values())
print(f"samples {S}  warp-instructions {N}")
for line, (s, n, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{line:>5} {100.0 * s / max(S, 1):5.1f}% {100.0 * n / max(N, 1):5.1f}%i  {src.strip()[:90]}")
