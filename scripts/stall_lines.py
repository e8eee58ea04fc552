"""Warp-stall samples per CUDA source line from `ncu -i R --page source --csv
--print-source cuda,sass --launch-count 1` exports (reports captured with
--import-source on and -lineinfo builds): the top lines of each kernel with
their three largest stall reasons.

  python scripts/stall_lines.py gpurun_out/reps/*_src.csv > profiles/<tag>_stall_lines.txt
"""
import collections
import csv
import os
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def lines_of(path, top=12):
    rows = list(csv.reader(open(path)))
    heads = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not heads:
        return None
    hi = heads[0]
    hdr = rows[hi]
    fn = [r for r in rows[:hi] if r and r[0] in ("Function Name", "Kernel Name")]
    stalls = [(k, hdr.index(k)) for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
    agg, det, src = collections.Counter(), collections.defaultdict(collections.Counter), {}
    end = heads[1] if len(heads) > 1 else len(rows)
    for r in rows[hi + 1:end]:
        if len(r) < 10 or r[0] == "":
            continue  # SASS rows under a source line
        try:
            ln = int(r[0])
        except ValueError:
            continue
        src[ln] = r[1]
        agg[ln] += num(r[4])
        for k, i in stalls:
            det[ln][k] += num(r[i])
    tot = sum(agg.values()) or 1
    out = [f"## {os.path.basename(path)[:-8]}: {fn[0][1][:110] if fn else ''} ({tot} samples)"]
    for ln, s in agg.most_common(top):
        why = ", ".join(f"{k[6:]}={v}" for k, v in det[ln].most_common(3) if v)
        out.append(f"{100 * s / tot:5.1f}%  L{ln}: {src.get(ln, '').strip()[:90]}  [{why}]")
    return "\n".join(out)


print("# ncu source-level warp-stall samples per CUDA line (top 12), --set full "
      "--import-source on, first captured launch of each report")
for f in sorted(sys.argv[1:]):
    block = lines_of(f)
    if block:
        print()
        print(block)
