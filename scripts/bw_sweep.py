"""Achieved HBM bandwidth of every state-vector kernel at large widths
(BASELINE config 4: gate + expectation roofline at 26-32 qubits).

Each kernel is timed with CUDA events on the state's stream (torch stream
handed to the engine), median over repeats; achieved = algorithmic bytes /
time, fraction = achieved / MEASURED_PEAKS.json hbm_gbs.

  python scripts/bw_sweep.py [n ...] [--f32]
"""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle.oracle import random_hamiltonian  # noqa: E402  (fixture generator only)
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def timed(stream, fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e-3


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    f32 = "--f32" in sys.argv
    widths = [int(a) for a in args] or [26, 28, 30]
    P = peak()
    V.init(0)
    stream = torch.cuda.Stream()
    out = []
    for n in widths:
        amp = 8 if f32 else 16
        S = (1 << n) * amp
        psi = V.StateVector(n, dtype="f32" if f32 else "f64")
        psi.set_stream(stream.cuda_stream)
        with torch.cuda.stream(stream):
            V.apply_circuit(psi, [V.Gate.ry(0.3, q) for q in range(n)])  # dense state
            rows = []

            def gate(g, alg):
                t = timed(stream, lambda: V.apply_gate(psi, g))
                rows.append((g.kind, g.wires, alg, t))

            for q in sorted({0, 1, n // 2, n - 5, n - 3, n - 2, n - 1}):
                gate(V.Gate.ry(0.1, q), 2 * S)
            gate(V.Gate.pauli_x(n // 3), 2 * S)
            for c, t_ in [(0, 1), (n // 2, n // 2 + 1), (n - 2, n - 1), (n - 1, 0)]:
                gate(V.Gate.cnot(c, t_), S)
            gate(V.Gate.double_excitation(0.2, 0, 1, 2, 3), S // 4)
            gate(V.Gate.double_excitation(0.2, n - 4, n - 3, n - 2, n - 1), S // 4)
            gate(V.Gate.single_excitation(0.2, 2, n - 2), S)
            plans = {}
            for name, h, groups in [
                ("zsum", V.build_z_sum(n), 1),
                ("tfim", V.build_tfim(n, 1.0, 1.0), n + 1),
            ]:
                t = timed(stream, lambda: V.expectation(psi, h), reps=3)
                rows.append(("expect:" + name, (), S * groups, t))
                plans["expect:" + name] = V.expectation_plan(h, "f32" if f32 else "f64")
            import random

            rh = random_hamiltonian(random.Random(20260804), n, 32)
            hv = V.canonicalize(V.QubitHamiltonian(n, [V.PauliTerm(c, a) for c, a in rh.terms]))
            flips = set()
            for term in hv.terms:
                f = sum(1 << (n - 1 - q) for q, a in term.axes if a in (1, 2))
                flips.add(f)
            t = timed(stream, lambda: V.expectation(psi, hv), reps=3)
            rows.append(("expect:random32", (), S * len(flips | {0}), t))
            plans["expect:random32"] = V.expectation_plan(hv, "f32" if f32 else "f64")
        for kind, wires, alg, t in rows:
            gbs = alg / t / 1e9
            rec = {"n": n, "dtype": "f32" if f32 else "f64", "kernel": kind, "wires": list(wires), "alg_bytes": alg,
                   "ms": t * 1e3, "GBps": gbs, "frac_of_measured_peak": gbs / P}
            if kind in plans:  # alg_bytes = S per flip group (+ diagonal); the engine reads the state per pass
                rec["plan"] = plans[kind]
                rec["pass_GBps"] = plans[kind]["state_passes"] * S / t / 1e9
                rec["pass_frac"] = rec["pass_GBps"] / P
            out.append(rec)
            print(json.dumps(rec), flush=True)
        del psi
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
