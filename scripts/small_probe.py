"""Latency of the small-register VQE path (n <= 8) through the public API:
run_scaling_study / run_vqe at HEA(2), 5 Adam iterations; repeated calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V
V.init(0)
for n in (4, 6, 8):
    for method in ("shift", "adjoint"):
        ts = []
        for rep in range(8):
            t0 = time.perf_counter()
            r = V.run_scaling_study(V.ScalingConfig(qubits=[n], method=method))[0]
            ts.append((time.perf_counter() - t0, r["runtime_seconds"]))
        print(n, method, " ".join(f"{a*1e3:.3f}/{b*1e3:.3f}" for a, b in ts), flush=True)
