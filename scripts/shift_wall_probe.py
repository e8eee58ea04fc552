"""Wall vs reported runtime of repeated shift-method scaling studies at one width:
python scripts/shift_wall_probe.py n [iterations]."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V
n = int(sys.argv[1])
it = int(sys.argv[2]) if len(sys.argv) > 2 else 5
V.init(0)
for rep in range(3):
    t0 = time.perf_counter()
    r = V.run_scaling_study(V.ScalingConfig(qubits=[n], method="shift", iterations=it, force=n > 26))[0]
    print(n, it, f"wall {time.perf_counter() - t0:.4f} s runtime {r['runtime_seconds']:.4f} s", flush=True)
