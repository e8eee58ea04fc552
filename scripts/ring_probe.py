"""k_tile ring-size check: fused circuits (apply_circuit) vs one launch per
gate (apply_gate) on the same state, permutation-only and mixed passes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2601_09951_b200 import vqeforge as V

V.init(0)
for n in [int(a) for a in sys.argv[1:]] or [20, 24, 28]:
    base = [V.Gate.ry(0.3 + 0.01 * q, q) for q in range(n)]
    tests = {
        "perm": [V.Gate.pauli_x(0), V.Gate.pauli_x(0), V.Gate.cnot(3, n - 1), V.Gate.cnot(3, n - 1)],
        "perm2": [V.Gate.cnot(q, q + 1) for q in range(n - 1)],
        "mixed": [V.Gate.ry(0.2, q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)],
    }
    for name, gs in tests.items():
        a = V.StateVector(n)
        V.apply_circuit(a, base)
        b = V.StateVector(n)
        V.apply_circuit(b, base)
        V.apply_circuit(a, gs)
        for g in gs:
            V.apply_gate(b, g)
        d = np.max(np.abs(a.amplitudes - b.amplitudes))
        print(f"{os.environ.get('TAG','')} n={n} {name}: max diff {d:.3e}", flush=True)
        del a, b
