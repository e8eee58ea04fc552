"""Tile fusion: one HEA layer (RY on every wire + CNOT chain) as a fused
apply_circuit vs the same gates one launch each; also checks they agree."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2601_09951_b200 import vqeforge as V

V.init(0)
s = torch.cuda.Stream()
for n in [20, 26, 30]:
    gates = [V.Gate.ry(0.1 * (q + 1), q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
    a, b = V.StateVector(n), V.StateVector(n)
    a.set_stream(s.cuda_stream); b.set_stream(s.cuda_stream)
    def t_of(fn, reps=3):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); fn(); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)
    tf = t_of(lambda: V.apply_circuit(a, gates))
    tu = t_of(lambda: [V.apply_gate(b, g) for g in gates])
    S = (1 << n) * 16
    ok = ""
    if n <= 26:
        ok = f"max|diff|={np.max(np.abs(a.amplitudes - b.amplitudes)):.2e}"
    print(f"n={n}: fused {tf:.3f} ms  unfused {tu:.3f} ms  speedup {tu / tf:.2f}x  "
          f"fused eff. {2 * S * len(gates) / (tf * 1e-3) / 1e9:.0f} GB/s-equivalent  {ok}", flush=True)
    del a, b
    torch.cuda.empty_cache()
