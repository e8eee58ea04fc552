"""CPU, world_size 2 over gloo: the N > 1 orchestration of the bond-sharded
PES (paper_2601_09951_b200/dist.py) — slices, max-over-ranks timing and the
rank-ordered gather reproduce the single-process sweep bit for bit.  Each
rank's slice is computed by the CPU oracle here (test infrastructure); on
the GPU box the same function runs the engine (bench.py)."""
from __future__ import annotations

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_points, iters, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from oracle.oracle import load_orc
    from paper_2601_09951_b200 import dist as D
    from paper_2601_09951_b200 import vqeforge as V

    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = load_orc()

    def run_slice(cfg):
        lo, hi = D.rank_slice(cfg.n_points, cfg.n_chunks, cfg.chunk_index)
        full = orc.run_sweep(cfg.d_min, cfg.d_max, cfg.n_points, max_iter=cfg.adam.max_iterations)
        return [(float(full["bond"][i]), float(full["energy"][i]), int(full["iterations"][i])) for i in range(lo, hi)]

    cfg = V.SweepConfig(d_min=0.3, d_max=2.5, n_points=n_points, adam=V.AdamConfig(max_iterations=iters))
    pts = D.sharded_sweep(cfg, rank, world, run_slice, dist)
    t = D.max_over_ranks(0.5 + rank, dist)
    if rank == 0:
        out.put((pts, t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_points", [7, 10])
def test_sharded_sweep_gloo_world2(n_points):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_points, 15, q)) for r in range(2)]
    for p in procs:
        p.start()
    pts, t = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    from oracle.oracle import load_orc

    full = load_orc().run_sweep(0.3, 2.5, n_points, max_iter=15)
    want = [(float(full["bond"][i]), float(full["energy"][i]), int(full["iterations"][i])) for i in range(n_points)]
    assert pts == want  # bitwise: grid order, values, iteration counts
    assert t == 1.5  # max over ranks


def test_rank_slices_partition_the_grid():
    sys.path.insert(0, ROOT)
    from paper_2601_09951_b200 import dist as D

    for world in [1, 2, 3, 4, 8]:
        cover = []
        for r in range(world):
            lo, hi = D.rank_slice(100, world, r)
            cover += list(range(lo, hi))
        assert cover == list(range(100))
    assert [hi - lo for lo, hi in (D.rank_slice(100, 8, r) for r in range(8))] == [13, 13, 13, 13, 12, 12, 12, 12]
