"""BASELINE config 3: the qubit-scaling study (run_scaling_study,
sweep.hpp:265-307: HEA(2 layers), TFIM J=h=1, 5 Adam iterations, lr 0.05,
theta0 = 0.1) on one B200 vs the reference's own CPU path (oracle/_ref,
single-threaded as the reference's state-vector kernels are), plus a random
32-term Pauli sum (test_helpers.hpp:28-59 semantics) variant.

  python scripts/bench_scaling.py [--ref-max 16] [--gpu-max 26]
Prints one JSON record per (width, engine).
"""
from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import load_ref, random_hamiltonian  # noqa: E402
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-max", type=int, default=16)
    ap.add_argument("--gpu-max", type=int, default=26)
    args = ap.parse_args()
    V.init(0)
    ref = load_ref()
    widths = [w for w in (4, 8, 12, 14, 16, 18, 20, 22, 24, 26) if w <= args.gpu_max]
    # warm-up (context, allocations, kernel attributes)
    V.run_scaling_study(V.ScalingConfig(qubits=[8], iterations=1))
    V.run_scaling_study(V.ScalingConfig(qubits=[8], iterations=1, method="adjoint"))
    for n in widths:
        for method in ("shift", "adjoint"):
            # a first run at each width pays one-time costs (state allocations
            # from the pool, kernel attributes); the second run is reported
            V.run_scaling_study(V.ScalingConfig(qubits=[n], method=method, force=n > 26))
            t0 = time.perf_counter()
            rec = V.run_scaling_study(V.ScalingConfig(qubits=[n], method=method, force=n > 26))[0]
            wall = time.perf_counter() - t0
            print(json.dumps({"config": "tfim-hea2", "engine": f"b200-{method}", "n": n, "runtime_s": rec["runtime_seconds"],
                              "wall_s": wall, "final_energy": rec["final_energy"], "iterations": rec["iterations_run"]}),
                  flush=True)
        if ref is not None and n <= args.ref_max:
            rec = ref.run_scaling_study([n])[0]
            print(json.dumps({"config": "tfim-hea2", "engine": "reference-cpu-1thread", "n": n,
                              "runtime_s": rec["runtime_seconds"], "final_energy": rec["final_energy"],
                              "iterations": rec["iterations_run"]}), flush=True)
    # random 32-term Pauli sum, HEA(2), 5 iterations
    for n in [w for w in widths if w <= 24]:
        h = random_hamiltonian(random.Random(20260804), n, 32)
        hv = V.canonicalize(V.QubitHamiltonian(n, [V.PauliTerm(c, a) for c, a in h.terms]))
        cfg = V.AdamConfig(learning_rate=0.05, max_iterations=5)
        init = [0.1] * (2 * n)
        for method in ("shift", "adjoint"):
            V.run_vqe(hv, V.AnsatzSpec.hardware_efficient(2), cfg, init, method=method)  # warm-up at this width
            t0 = time.perf_counter()
            r = V.run_vqe(hv, V.AnsatzSpec.hardware_efficient(2), cfg, init, method=method)
            print(json.dumps({"config": "random32-hea2", "engine": f"b200-{method}", "n": n,
                              "runtime_s": time.perf_counter() - t0, "final_energy": r.energy}), flush=True)
        if ref is not None and n <= min(args.ref_max, 14):
            from oracle.oracle import Ham
            hr = Ham(n, [(t.coefficient, t.axes) for t in hv.terms])
            t0 = time.perf_counter()
            r = ref.run_vqe(hr, kind=1, layers=2, lr=0.05, max_iter=5, init=init)
            print(json.dumps({"config": "random32-hea2", "engine": "reference-cpu-1thread", "n": n,
                              "runtime_s": time.perf_counter() - t0, "final_energy": r["energy"]}), flush=True)


if __name__ == "__main__":
    main()
