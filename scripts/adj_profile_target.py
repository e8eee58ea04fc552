"""One 26-qubit adjoint VQE iteration (HEA 2 layers, TFIM) for ncu launch lists."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2601_09951_b200 import vqeforge as V
V.init(0)
V.run_scaling_study(V.ScalingConfig(qubits=[26], iterations=1, method="adjoint"))
