"""Times the fused PES kernel at several iteration counts: the intercept is
the chemistry prologue, the slope the per-Adam-iteration latency."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_09951_b200 import vqeforge as V

V.init(0)
s = torch.cuda.Stream()
res = []
for iters in [0, 1, 10, 50, 100, 200]:
    plan = V.PesPlan(V.SweepConfig(adam=V.AdamConfig(max_iterations=iters)))
    for _ in range(5):
        plan.launch(s.cuda_stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in ev:
        a.record(s); plan.launch(s.cuda_stream); b.record(s)
    torch.cuda.synchronize()
    t = statistics.median(a.elapsed_time(b) for a, b in ev) * 1e3
    res.append((iters, t))
    print(f"iters={iters:4d}  {t:8.1f} us", flush=True)
(i0, t0), (i1, t1) = res[0], res[-1]
print(f"prologue ~{t0:.1f} us, per-iteration ~{(t1 - t0) / (i1 - i0) * 1e3:.1f} ns")
