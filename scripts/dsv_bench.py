"""BASELINE config 5 machinery on one B200: an n-qubit state split over
`world` virtual shards (vqf_dsv_* through paper_2601_09951_b200/dsv.py:
shards in this process, global-qubit swaps as in-place device swaps) vs the
single-state engine, for one hardware-efficient layer (apply_circuit: fused
local runs + lazy swaps) and a TFIM expectation.  The exchange here is an
HBM swap, not NVLink; the point is the sharded path's structure and
overhead (swaps per layer, bytes exchanged).

  python scripts/dsv_bench.py [n] [world]
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_09951_b200 import vqeforge as V  # noqa: E402
from paper_2601_09951_b200.dsv import DistributedStateVector  # noqa: E402


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dtype = sys.argv[3] if len(sys.argv) > 3 else "f64"
    V.init(0)
    layer = [(1, 0.1 * (q + 1), [q]) for q in range(n)] + [(2, 0.0, [q, q + 1]) for q in range(n - 1)]
    tfim = V.build_tfim(n, 1.0, 1.0)
    terms = [(t.coefficient, t.axes) for t in tfim.terms]
    d = DistributedStateVector(n, world, dtype=dtype)
    s0 = d.stats()["swaps"]
    t_layer_d = wall(lambda: d.apply_circuit(layer))  # 4 layers applied (1 warm-up + 3 timed)
    swaps_layer = (d.stats()["swaps"] - s0) / 4
    s0 = d.stats()["swaps"]
    t_exp_d = wall(lambda: d.expectation(terms))
    swaps_exp = (d.stats()["swaps"] - s0) / 4
    e_d = d.expectation(terms)
    del d
    torch.cuda.empty_cache()
    single = V.StateVector(n, dtype=dtype)
    gates = [V.Gate(k, a, tuple(w)) for k, a, w in layer]
    t_layer_s = wall(lambda: V.apply_circuit(single, gates))
    t_exp_s = wall(lambda: V.expectation(single, tfim))
    e_s = V.expectation(single, tfim)
    print(json.dumps({"n": n, "world": world, "dtype": dtype, "shard_qubits": n - (world.bit_length() - 1),
                      "hea_layer_s": {"sharded": t_layer_d, "single": t_layer_s, "swaps": swaps_layer},
                      "tfim_expectation_s": {"sharded": t_exp_d, "single": t_exp_s, "swaps": swaps_exp},
                      "tfim_energy": {"sharded": e_d, "single": e_s, "abs_diff": abs(e_d - e_s)},
                      "note": "virtual ranks on one GPU (config-5 sizes fit one B200 in fp32 at n = 34 / fp64 at "
                              "n = 33); swaps are in-place HBM swaps, not NVLink; wall clock, median of 3; 4 HEA "
                              "layers applied to both states before the energies"}))


if __name__ == "__main__":
    main()
