"""Small, deterministic workloads for ncu captures (run under gpurun).

  python scripts/prof_targets.py pes        # fused PES kernel, 3 launches
  python scripts/prof_targets.py gates N    # RY / CNOT / DE on an N-qubit fp64 state
  python scripts/prof_targets.py expect N   # TFIM expectation (diag + N flip groups)
  python scripts/prof_targets.py hea N [f32]      # two fused HEA layers (k_tile passes)
  python scripts/prof_targets.py expect N [f32]   # (dtype option for both)
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_09951_b200 import vqeforge as V  # noqa: E402


def main():
    what = sys.argv[1]
    V.init(0)
    if what == "pes":
        plan = V.PesPlan(V.SweepConfig())
        for _ in range(3):
            plan.launch()
        rep = plan.read()
        assert rep.all_ok
    elif what == "gates":
        n = int(sys.argv[2])
        psi = V.StateVector(n)
        # per-gate kernels (apply_gate), not the fused tile path
        for g in [V.Gate.ry(0.3, q) for q in (0, 1, n // 2, n - 2, n - 1)] + [
                V.Gate.cnot(0, 1), V.Gate.cnot(n - 2, n - 1), V.Gate.double_excitation(0.4, 0, 1, 2, 3),
                V.Gate.double_excitation(0.4, n - 4, n - 3, n - 2, n - 1), V.Gate.single_excitation(0.4, 2, n - 2)]:
            V.apply_gate(psi, g)
    elif what == "expect":
        n = int(sys.argv[2])
        psi = V.StateVector(n, dtype=sys.argv[3] if len(sys.argv) > 3 else "f64")
        V.apply_circuit(psi, [V.Gate.ry(0.3, q) for q in range(n)])
        print(V.expectation(psi, V.build_tfim(n, 1.0, 1.0)))
        print(V.expectation(psi, V.build_z_sum(n)))
    elif what == "hea":
        n = int(sys.argv[2])
        psi = V.StateVector(n, dtype=sys.argv[3] if len(sys.argv) > 3 else "f64")
        layer = [V.Gate.ry(0.1 * (q + 1), q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
        for _ in range(2):
            V.apply_circuit(psi, layer)
    else:
        raise SystemExit(f"unknown target {what}")


if __name__ == "__main__":
    main()
