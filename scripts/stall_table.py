"""Per-instruction warp-stall table from an `ncu --page source --csv
--print-source sass` export: totals by stall reason and the hottest
instructions.  usage: stall_table.py file.csv [top] [kernel_section]"""
import csv
import sys

allrows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # kernel section index
starts = [i for i, r in enumerate(allrows) if r and r[0] == "Kernel Name"]
starts.append(len(allrows))
rows = allrows[starts[which]:starts[which + 1]]
print(rows[0][1] if len(rows[0]) > 1 else "")
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    per = {k: int(r[ix[k]] or 0) for k in reasons}
    for k in reasons:
        tot[k] += per[k]
    data.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip(), per))
S = sum(d[0] for d in data)
print("total samples", S)
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print(f"  {k:28s} {v:7d} {100.0 * v / max(S, 1):5.1f}%")
print()
for s, a, src, per in sorted(data, key=lambda x: -x[0])[:top]:
    main = ", ".join(f"{k[6:]}={v}" for k, v in sorted(per.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{s:6d} {a} {src[:60]:60s} {main}")
