"""Repeated parameter-shift scaling-study runs at small/mid widths (ms per
run): python scripts/shift_repeat_probe.py n [n ...]."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V
V.init(0)
tag = "noshare" if os.environ.get("VQF_NO_SHARED_PREFIX") else "shared"
for n in [int(a) for a in sys.argv[1:]]:
    ts = []
    for rep in range(10):
        r = V.run_scaling_study(V.ScalingConfig(qubits=[n], method="shift"))[0]
        ts.append(r["runtime_seconds"] * 1e3)
    print(tag, n, " ".join(f"{t:.2f}" for t in ts), flush=True)
