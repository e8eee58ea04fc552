"""One-process-per-GPU orchestration for the bond-sharded PES (BASELINE
config 2).  torch.distributed is plumbing only: the data path has no
collective; ranks own disjoint split_chunks slices of the global bond grid
(sweep.hpp:93-107) and meet once to reduce timings and gather results.
"""
from __future__ import annotations

import os
from typing import Callable, List, Optional, Sequence, Tuple

from . import vqeforge as V


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def rank_slice(n_points: int, world: int, rank: int) -> Tuple[int, int]:
    """This rank's [begin, end) of the global grid — the same split the C ABI
    applies for vqf_sweep_config.chunk_index / n_chunks."""
    return V.split_chunks(n_points, world)[rank]


def max_over_ranks(value: float, dist=None, device: Optional[str] = None) -> float:
    """Whole-job time = the slowest rank (timing rule: max over ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_points(local: Sequence, dist=None) -> List:
    """Concatenates every rank's points in rank order (= grid order, since
    slices are contiguous and ascending)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, list(local))
    return [p for part in parts for p in part]


def sharded_sweep(config: V.SweepConfig, rank: int, world: int,
                  run_slice: Callable[[V.SweepConfig], Sequence], dist=None) -> List:
    """Runs this rank's slice with `run_slice` (the engine: a PesPlan or
    run_sweep on this rank's GPU) and gathers the full, grid-ordered list."""
    cfg = V.SweepConfig(d_min=config.d_min, d_max=config.d_max, n_points=config.n_points, workers=1,
                        adam=config.adam, devices=config.devices, chunk_index=rank, n_chunks=world)
    return gather_points(run_slice(cfg), dist)
