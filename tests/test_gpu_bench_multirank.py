"""bench.py's N > 1 path (BASELINE config 2: the bond grid sharded over
ranks, max-over-ranks timing, rank-ordered gather, parity against the
reference fixture) run for real under torchrun with two ranks.  A one-GPU box
cannot host two NCCL ranks, so VQF_BENCH_SHARE_GPU=1 puts both on cuda:0 over
gloo; everything else is the path the driver's multi-GPU run takes."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _torchrun(args, nproc=2):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py"] + args
    env = dict(os.environ, VQF_BENCH_SHARE_GPU="1")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("world", [2, 8])
def test_bench_ranks_sharded_pes(world):
    lines = _torchrun(["--gpus", str(world), "--steps", "3", "--warmup", "3", "--gate-qubits", "0"], nproc=world)
    assert len(lines) == 1  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == world and f"over {world} GPU" in line["config"]["parallelism"]
    par = line["parity"]
    assert par["bond_grid_bitwise"] and par["iterations_equal"] and par["all_ok"] and par["e2e_equals_value_run"]
    assert par["max_abs_dE_vs_reference"] < 1e-10
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] >= 3


def test_bench_reference_arm_two_ranks():
    lines = _torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
