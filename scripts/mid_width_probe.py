"""Config-3 widths: run_scaling_study (HEA(2), TFIM, 5 iterations) per
engine, 9 repetitions each (median / min / max wall of the library call),
beside the reference's single-threaded run_scaling_study (oracle/_ref).
  python scripts/mid_width_probe.py [widths...]"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import load_ref  # noqa: E402
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402


def main():
    widths = [int(x) for x in sys.argv[1:]] or [4, 5, 6, 8, 10, 12, 13, 14, 16]
    V.init(0)
    ref = load_ref()
    for n in widths:
        for engine in ("", "warp", "block", "hbm"):
            if engine == "warp" and n > 5:
                continue
            os.environ["VQF_ENGINE"] = engine
            for method in ("shift", "adjoint"):
                try:
                    V.run_scaling_study(V.ScalingConfig(qubits=[n], method=method))
                except Exception as e:  # engine does not hold this width
                    print(json.dumps({"n": n, "engine": engine or "auto", "method": method, "error": str(e)[:80]}), flush=True)
                    break
                ts, rts = [], []
                for _ in range(9):
                    t0 = time.perf_counter()
                    rec = V.run_scaling_study(V.ScalingConfig(qubits=[n], method=method))[0]
                    ts.append(time.perf_counter() - t0)
                    rts.append(rec["runtime_seconds"])
                print(json.dumps({"n": n, "engine": engine or "auto", "method": method,
                                  "runtime_median_s": statistics.median(rts), "runtime_min_s": min(rts),
                                  "runtime_max_s": max(rts), "wall_median_s": statistics.median(ts),
                                  "final_energy": rec["final_energy"]}), flush=True)
        os.environ["VQF_ENGINE"] = ""
        if ref is not None and n <= 14:
            reps = 5 if n <= 10 else 1
            rts = [ref.run_scaling_study([n])[0]["runtime_seconds"] for _ in range(reps)]
            print(json.dumps({"n": n, "engine": "reference-cpu-1thread", "runtime_median_s": statistics.median(rts),
                              "runtime_min_s": min(rts), "runtime_max_s": max(rts)}), flush=True)


if __name__ == "__main__":
    main()
