import os, sys
sys.path.insert(0, "/root/repo")
from paper_2601_09951_b200 import vqeforge as V
V.init(0)
n = 26
gates = [V.Gate.ry(0.1 * (q + 1), q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
a = V.StateVector(n)
V.apply_circuit(a, gates)
