"""Parameter-shift run_scaling_study at n = 16 before and after a large
(config-4 sized) state has been created and freed in the same process, as
in bench.py: per-run runtime plus the CUDA runtime calls that dominate the
slow runs (torch profiler, CPU + CUDA activity).
usage: python scripts/shift_alloc_probe.py [n] [big_n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

V.init(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
big = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = V.ScalingConfig(qubits=[n], method="shift")


def runs(tag, k=7, profile=False, each=False):
    ts = []
    for rep in range(k):
        t0 = time.perf_counter()
        if each:
            acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
            with torch.profiler.profile(activities=acts) as prof:
                rt = V.run_scaling_study(cfg)[0]["runtime_seconds"]
            tot = {}
            ksum = 0.0
            for e in prof.events():
                if e.name.startswith("cuda"):
                    c, t = tot.get(e.name, (0, 0.0))
                    tot[e.name] = (c + 1, t + e.cpu_time_total / 1e3)
                if e.device_type == torch.autograd.DeviceType.CUDA:
                    ksum += e.device_time / 1e3
            print(f"  {tag} run {rep}: {rt*1e3:.2f} ms, device-sum {ksum:.2f} ms,",
                  sorted(((k2, c, round(t, 3)) for k2, (c, t) in tot.items()), key=lambda x: -x[2])[:4], flush=True)
        else:
            rt = V.run_scaling_study(cfg)[0]["runtime_seconds"]
        ts.append((rt, time.perf_counter() - t0))
    print(tag, " ".join(f"{a*1e3:.2f}" for a, _ in ts), flush=True)
    if profile:
        acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
        with torch.profiler.profile(activities=acts) as prof:
            V.run_scaling_study(cfg)
        tot = {}
        for e in prof.events():
            if e.name.startswith("cuda"):
                c, t = tot.get(e.name, (0, 0.0))
                tot[e.name] = (c + 1, t + e.cpu_time_total / 1e3)
        print(tag, "runtime calls:", sorted(((k, c, round(t, 3)) for k, (c, t) in tot.items()), key=lambda x: -x[2])[:8],
              flush=True)


if os.environ.get("AFTER_BENCH"):
    import bench
    bench.configs_3_4(V, torch, 0, 30, 3, 3, 6548.2, False, 0)
    runs("after-bench")
    runs("after-bench-prof", k=5, each=True)
if os.environ.get("AFTER_N26"):
    for nq in (20, 24, 26):
        h = V.build_tfim(nq, 1.0, 1.0)
        for method in ("shift", "adjoint"):
            c = V.AdamConfig(learning_rate=0.05, max_iterations=1)
            for _ in range(2):
                V.run_vqe(h, V.AnsatzSpec.hardware_efficient(2), c, [0.1] * (2 * nq), method=method)
    if os.environ.get("SLEEP"):
        time.sleep(float(os.environ["SLEEP"]))
    smi = None
    if os.environ.get("SMI"):
        import subprocess
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                                "--format=csv,noheader", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    runs("after-n26")
    if smi is not None:
        smi.terminate()
        print("smi:", " | ".join(l.strip() for l in smi.stdout.read().splitlines()[:40]))
    runs("after-n26-prof", k=5, each=True)
runs("fresh", profile=True)
s = V.StateVector(big)
V.apply_circuit(s, [V.Gate.ry(0.3, q) for q in range(big)])
V.expectation(s, V.build_tfim(big, 1.0, 1.0))
del s
runs("after-big", profile=True)
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
del x
runs("after-torch", k=10, each=True)
