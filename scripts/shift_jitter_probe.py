"""Host-side view of parameter-shift run_vqe jitter at n = 16: per-run wall
time and device kernel time (torch profiler over CUPTI sees every kernel)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

V.init(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = V.ScalingConfig(qubits=[n], method="shift")
V.run_scaling_study(cfg)
walls = []
for rep in range(8):
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        rt = V.run_scaling_study(cfg)[0]["runtime_seconds"]
        w = time.perf_counter() - t0
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ktime = sum(e.device_time for e in ev) / 1e3
    kinds = {}
    for e in ev:
        kinds[e.name[:40]] = kinds.get(e.name[:40], 0) + 1
    print(f"rep {rep}: runtime {rt*1e3:.2f} ms wall {w*1e3:.2f} ms kernels {len(ev)} device-sum {ktime:.2f} ms", flush=True)
print(sorted(kinds.items(), key=lambda x: -x[1])[:12])
