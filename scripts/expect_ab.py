"""Median device time of expectation() for TFIM and a random 32-term sum on
a random-ish state (RY layer) at the given widths: A/B of expectation
kernels (TAG env names the build)."""
import os, random, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_09951_b200 import vqeforge as V
from oracle.oracle import random_hamiltonian

V.init(0)
s = torch.cuda.Stream()
for n in [int(a) for a in sys.argv[1:]] or [28, 30]:
    dt = os.environ.get("DTYPE", "f64")
    psi = V.StateVector(n, dtype=dt)
    psi.set_stream(s.cuda_stream)
    V.apply_circuit(psi, [V.Gate.ry(0.1 * (q + 1), q) for q in range(n)])
    hs = {"tfim": V.build_tfim(n, 1.0, 1.0)}
    for name, h in hs.items():
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); e = V.expectation(psi, h); e1.record(s); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{os.environ.get('TAG', '')} {dt} n={n} {name} passes={V.expectation_plan(h, dt)['state_passes']}: {statistics.median(ts[2:]):.3f} ms  E={e!r}", flush=True)
    del psi
    torch.cuda.empty_cache()
