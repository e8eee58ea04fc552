"""Generates the committed golden fixtures in tests/golden/ from the
reference's own CPU path (oracle/_ref/libvqf_ref.so = the unmodified
/root/reference/proj/include headers compiled against oracle/eigen_shim).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The fixtures are small JSON files; the GPU box reads only these files.
Floats are stored with repr() (17 significant digits, bit-exact round trip).
"""
from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Ham, Reference, random_hamiltonian, random_state  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def ham_json(h: Ham):
    return {"n_qubits": h.n_qubits, "text": h.to_text()}


def cplx_list(a):
    return [[float(x.real), float(x.imag)] for x in a]


def main():
    R = Reference()

    # 1. H2 Hamiltonians (chem.hpp:473) on a spread of bonds + the defaults grid.
    bonds = [0.1, 0.3, 0.5, 0.7414, 0.9, 1.1, 1.2, 1.6, 2.0, 2.6, 3.0] + list(R.bond_grid(0.1, 3.0, 100)[::11])
    h2 = {repr(float(d)): ham_json(R.build_h2_hamiltonian(float(d))) for d in bonds}
    hf = {repr(float(d)): R.hartree_fock(float(d)) for d in bonds}
    e0 = {repr(float(d)): R.exact_ground_energy(R.build_h2_hamiltonian(float(d))) for d in bonds}
    with open(os.path.join(OUT, "h2_hamiltonians.json"), "w") as f:
        json.dump({"hamiltonians": h2, "hartree_fock": hf, "exact_ground_energy": e0}, f, indent=1)

    # 2. Default PES (sweep.hpp:128 with SweepConfig{}), fixed 200 iterations,
    #    plus tol mode (1e-8, <= 5000).
    pes = R.run_sweep()
    tol = R.run_sweep(max_iter=5000, tol=1e-8)
    with open(os.path.join(OUT, "pes_default.json"), "w") as f:
        json.dump({
            "config": {"d_min": 0.1, "d_max": 3.0, "n_points": 100, "max_iterations": 200},
            "bond": [float(x) for x in pes["bond"]],
            "energy": [float(x) for x in pes["energy"]],
            "theta": [float(x) for x in pes["theta"]],
            "iterations": [int(x) for x in pes["iterations"]],
            "tol_mode": {"max_iterations": 5000, "gradient_tolerance": 1e-8,
                         "energy": [float(x) for x in tol["energy"]],
                         "theta": [float(x) for x in tol["theta"]],
                         "iterations": [int(x) for x in tol["iterations"]]},
        }, f, indent=1)

    # 3. run_vqe trajectories (vqe.hpp:194) at a few bonds, H2 ansatz.
    traj = {}
    for d in [0.5, 0.7414, 1.1, 2.6]:
        h = R.build_h2_hamiltonian(d)
        r = R.run_vqe(h)
        traj[repr(d)] = {"energy": r["energy"], "theta": [float(x) for x in r["theta"]],
                         "trajectory": [float(x) for x in r["trajectory"]],
                         "circuit_evaluations": r["circuit_evaluations"]}
    # HEA on TFIM / Z-sum / random Pauli sums, small widths (run_scaling_study semantics).
    hea = {}
    for n, kind in [(4, "tfim"), (5, "zsum"), (6, "tfim"), (8, "tfim")]:
        h = R.build_tfim(n, 1.0, 1.0) if kind == "tfim" else R.build_z_sum(n)
        r = R.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=5, init=[0.1] * (2 * n))
        hea[f"{kind}{n}"] = {"hamiltonian": ham_json(h), "layers": 2, "lr": 0.05, "max_iterations": 5,
                             "theta_init": 0.1, "energy": r["energy"], "theta": [float(x) for x in r["theta"]],
                             "trajectory": [float(x) for x in r["trajectory"]],
                             "circuit_evaluations": r["circuit_evaluations"]}
    with open(os.path.join(OUT, "vqe_runs.json"), "w") as f:
        json.dump({"h2": traj, "hea": hea}, f, indent=1)

    # 4. Gate and expectation cases on seeded random states (n = 4..10).
    rng = np.random.default_rng(20260802)
    pr = random.Random(20260804)
    cases = []
    for n in [4, 5, 6, 8, 10]:
        psi = random_state(rng, n)
        gates = []
        for _ in range(24):
            k = pr.randint(0, 3)
            ws = pr.sample(range(n), [1, 1, 2, 4][k])
            gates.append([k, pr.uniform(-3.14, 3.14), ws])
        out = R.apply_gates(n, psi, [(g[0], g[1], g[2]) for g in gates])
        h = R.canonicalize(random_hamiltonian(pr, n, 12, real=True))
        cases.append({"n": n, "psi": cplx_list(psi), "gates": gates, "out": cplx_list(out),
                      "hamiltonian": ham_json(h), "expectation_out": R.expectation(n, out, h)})
    with open(os.path.join(OUT, "gates_expectation.json"), "w") as f:
        json.dump({"cases": cases}, f)

    # 5. Scaling study, Z-sum n = 4, 6 (test_sweep.cpp:195-212 configuration).
    sc = R.run_scaling_study([4, 6], layers=1, iterations=150, lr=0.1, z_sum=True)
    with open(os.path.join(OUT, "scaling_zsum.json"), "w") as f:
        json.dump({"config": {"qubits": [4, 6], "layers": 1, "iterations": 150, "learning_rate": 0.1,
                              "z_sum_mode": True, "theta_init": 0.1},
                   "records": [{k: v for k, v in r.items() if k != "runtime_seconds"} for r in sc]}, f, indent=1)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
