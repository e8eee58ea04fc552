"""Summarise the per-bond TIMELINE lines a -DVQF_STAGE_CLOCKS build prints
(globaltimer at kernel entry / loop start / loop end per CTA): spread of CTA
start times, prologue and loop durations, and the span of the whole launch.
usage: timeline.py stage.txt"""
import re
import statistics
import sys

rows = []
for line in open(sys.argv[1]):
    m = re.search(r"TIMELINE bond (\d+) sm (\d+) entry (\d+) prologue_ns (\d+) loop_ns (\d+) end (\d+)", line)
    if m:
        rows.append(tuple(int(x) for x in m.groups()))
if not rows:
    sys.exit("no TIMELINE lines")
# the last launch in the file (prof_targets runs several)
rows = rows[-100:]
t0 = min(r[2] for r in rows)
entry = [r[2] - t0 for r in rows]
pro = [r[3] for r in rows]
loop = [r[4] for r in rows]
end = [r[5] - t0 for r in rows]
q = lambda v: f"min {min(v) / 1e3:7.2f}  med {statistics.median(v) / 1e3:7.2f}  max {max(v) / 1e3:7.2f} us"
print("CTAs", len(rows), "distinct SMs", len({r[1] for r in rows}))
print("entry offset ", q(entry))
print("prologue     ", q(pro))
print("loop         ", q(loop))
print("end          ", q(end))
