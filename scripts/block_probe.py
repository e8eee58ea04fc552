"""One run_scaling_study per width on the shared-memory engine (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

V.init(0)
os.environ["VQF_ENGINE"] = "block"
for n in [int(x) for x in sys.argv[1:]] or [4, 8, 12, 13]:
    V.run_scaling_study(V.ScalingConfig(qubits=[n]))
