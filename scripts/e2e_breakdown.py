"""Where the end-to-end run_sweep time goes (GPU box): full C-ABI call with
and without trajectories vs the kernel's own device time, and the PesPlan
launch + read path.  usage: python scripts/e2e_breakdown.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
V.init(0)
for traj in ((False,) if os.environ.get("E2E_NOTRAJ") else (False, True)):
    buf = V.SweepBuffers(V.SweepConfig(), trajectories=traj)
    for _ in range(5):
        buf.run()
    t = []
    dev = []
    for _ in range(reps):
        t0 = time.perf_counter()
        buf.run()
        t.append(time.perf_counter() - t0)
        dev.append(buf.rep.device_seconds)
    t.sort()
    dev.sort()
    print(f"run_sweep traj={traj}: median {t[len(t) // 2] * 1e6:8.1f} us  min {t[0] * 1e6:8.1f} us  "
          f"device median {dev[len(dev) // 2] * 1e6:8.1f} us  wall-in-C {buf.rep.total_wall_seconds * 1e6:8.1f} us")
