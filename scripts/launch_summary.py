"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
[,dram__bytes_read.sum,dram__bytes_write.sum] --csv --log-file F):
python scripts/launch_summary.py F [n_first_launches]."""
import collections, csv, sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
k = collections.OrderedDict()
for r in csv.DictReader(lines[start:]):
    k.setdefault((r["ID"], r["Kernel Name"][:70], r["Grid Size"]), {})[r["Metric Name"]] = float(
        r["Metric Value"].replace(",", ""))
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, name, _), m in k.items():
    t = tot[name]
    t[0] += 1
    t[1] += m.get("gpu__time_duration.sum", 0)
    t[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
for name, (c, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{c:5d} {t / 1e6:10.3f} ms {b / 1e9:8.2f} GB {b / t if t else 0:7.0f} GB/s  {name}")
for (i, name, g), m in list(k.items())[: int(sys.argv[2]) if len(sys.argv) > 2 else 0]:
    print(i, name[:50], g, f"{m.get('gpu__time_duration.sum', 0) / 1e3:.1f} us",
          f"{(m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e6:.1f} MB")
