"""A/B of the adjoint backward sweep in a GF(2) frame (default) vs data
permutation passes (VQF_ADJ_NO_FRAME=1): one-iteration run_scaling_study."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V

V.init(0)
tag = "noframe" if os.environ.get("VQF_ADJ_NO_FRAME") else "frame"
for n in [int(a) for a in sys.argv[1:]] or [20, 24, 26]:
    cfg = V.ScalingConfig(qubits=[n], method="adjoint", iterations=1, force=n > 26)
    V.run_scaling_study(cfg)
    ts = sorted(V.run_scaling_study(cfg)[0]["runtime_seconds"] for _ in range(5))
    print(f"{tag} n={n}: {ts[2] * 1e3:.2f} ms  E={V.run_scaling_study(cfg)[0]['final_energy']!r}", flush=True)
