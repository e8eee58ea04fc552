"""Median device time of a fused HEA(2) circuit (apply_circuit) at several
widths; run twice with and without VQF_TILE_DENSE=1 for an A/B of the
fused-op kernels."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_09951_b200 import vqeforge as V

V.init(0)
s = torch.cuda.Stream()
for n in [int(a) for a in sys.argv[1:]] or [24, 26, 28]:
    gates = []
    for layer in range(int(os.environ.get("LAYERS", "2"))):
        gates += [V.Gate.ry(0.1 * (q + 1) + layer, q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
    dt = os.environ.get("DTYPE", "f64")
    a = V.StateVector(n, dtype=dt)
    a.set_stream(s.cuda_stream)
    ts = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); V.apply_circuit(a, gates); e1.record(s); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    plan = V.circuit_plan(n, gates, dt)
    S = (1 << n) * (16 if dt == "f64" else 8)
    med = statistics.median(ts[2:])
    print(f"{os.environ.get('TAG', '')} {dt} L{os.environ.get('LAYERS', '2')} n={n}: {med:.3f} ms (min {min(ts[2:]):.3f}) "
          f"{plan['passes']} passes, {2 * S * plan['passes'] / (med * 1e-3) / 1e9:.0f} GB/s", flush=True)
    del a
    torch.cuda.empty_cache()
