"""ncu target: one fused HEA layer (apply_circuit) at width n (default 28),
run 3 times; profile e.g. the 2nd pass of the last run with
  ncu --kernel-name regex:k_tile --launch-skip K --launch-count 1 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
dtype = sys.argv[2] if len(sys.argv) > 2 else "f64"
V.init(0)
gates = [V.Gate.ry(0.1 * (q + 1), q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
a = V.StateVector(n, dtype=dtype)
for _ in range(3):
    V.apply_circuit(a, gates)
print(V.circuit_plan(n, gates, dtype))
