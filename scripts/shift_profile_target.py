"""One parameter-shift VQE iteration (HEA 2 layers, TFIM) at width n for ncu
launch lists: python scripts/shift_profile_target.py [n]."""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2601_09951_b200 import vqeforge as V
n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
V.init(0)
V.run_scaling_study(V.ScalingConfig(qubits=[n], iterations=1, method="shift", force=n > 26))
