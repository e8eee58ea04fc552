"""Probe: does the L2 fetch granularity limit change the sector-sparse gates?

DoubleExcitation on the last four wires touches 2 of every 16 amplitudes
(2 of 8 sectors per 256 B); with a 64/128 B fetch granularity the DRAM moves
the whole neighbourhood.  Times sparse and dense gates at n with
cudaLimitMaxL2FetchGranularity = default, 32, 64, 128.

  python scripts/l2_gran_probe.py [n]
"""
from __future__ import annotations

import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

LIMIT_L2_FETCH = 5  # cudaLimitMaxL2FetchGranularity


def cudart():
    import nvidia.cuda_runtime as cr
    return ctypes.CDLL(os.path.join(cr.__path__[0], "lib", "libcudart.so.12"))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    rt = cudart()
    V.init(0)
    stream = torch.cuda.Stream()
    psi = V.StateVector(n)
    psi.set_stream(stream.cuda_stream)
    S = (1 << n) * 16
    gates = [
        ("DE_low", V.Gate.double_excitation(0.2, n - 4, n - 3, n - 2, n - 1), S // 4),
        ("DE_high", V.Gate.double_excitation(0.2, 0, 1, 2, 3), S // 4),
        ("SE_2_nm2", V.Gate.single_excitation(0.2, 2, n - 2), S),
        ("CNOT_low", V.Gate.cnot(n - 2, n - 1), S),
        ("CNOT_high", V.Gate.cnot(0, 1), S),
        ("RY_low", V.Gate.ry(0.1, n - 1), 2 * S),
        ("RY_mid", V.Gate.ry(0.1, n // 2), 2 * S),
    ]
    cur = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(cur), LIMIT_L2_FETCH)
    default = cur.value
    print(json.dumps({"default_l2_fetch_granularity": default}), flush=True)
    with torch.cuda.stream(stream):
        V.apply_circuit(psi, [V.Gate.ry(0.3, q) for q in range(n)])
        for gran in (default, 32, 64, 128):
            rc = rt.cudaDeviceSetLimit(LIMIT_L2_FETCH, ctypes.c_size_t(gran))
            rt.cudaDeviceGetLimit(ctypes.byref(cur), LIMIT_L2_FETCH)
            for name, g, alg in gates:
                ts = []
                for _ in range(7):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    V.apply_gate(psi, g)
                    b.record(stream)
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b) * 1e-3)
                t = statistics.median(ts)
                print(json.dumps({"n": n, "set": gran, "rc": rc, "got": cur.value, "gate": name, "ms": t * 1e3,
                                  "alg_GBps": alg / t / 1e9}), flush=True)


if __name__ == "__main__":
    main()
