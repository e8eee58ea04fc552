"""Distributed state vector (BASELINE config 5) on CPU: virtual ranks
(LocalComm) and world_size-2 gloo processes (TorchComm), local compute by
the oracle, checked against a single-state oracle run (amplitudes 1e-12,
energies 1e-10)."""
from __future__ import annotations

import os
import random
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.oracle import load_orc, random_hamiltonian, random_state  # noqa: E402


def circuit(pr, n, count):
    gates = []
    for _ in range(count):
        k = pr.randint(0, 3)
        ws = pr.sample(range(n), [1, 1, 2, 4][k])
        gates.append((k, pr.uniform(-3, 3), ws))
    # make sure global wires are exercised
    gates += [(1, 0.7, [0]), (2, 0.0, [0, n - 1]), (2, 0.0, [n - 2, 1]), (3, 0.4, [1, 0, n - 1, 3])]
    return gates


def run_case(dsv_cls, backend, comm, n, world, seed):
    orc = load_orc()
    rng = np.random.default_rng(seed)
    pr = random.Random(seed)
    psi = random_state(rng, n)
    d = dsv_cls(n, world, backend, comm)
    d.set_full(psi)
    gates = circuit(pr, n, 25)
    for k, a, w in gates:
        d.apply_gate(k, a, w)
    want = orc.apply_gates(n, psi, gates)
    got = d.local_amplitudes()
    nl = n - (world.bit_length() - 1)
    h = orc.canonicalize(random_hamiltonian(pr, n, 24))
    e_want = orc.expectation(n, want, h)
    e_got = d.expectation(h.terms)
    return want, got, nl, e_want, e_got, d.swaps_done


@pytest.mark.parametrize("world,n", [(2, 7), (4, 8), (8, 9), (4, 10)])
def test_dsv_virtual_ranks_match_single_state(world, n):
    from dsv_cpu_backend import CpuOracleBackend
    from paper_2601_09951_b200.dsv import DistributedStateVector, LocalComm

    want, got, nl, e_want, e_got, swaps = run_case(DistributedStateVector, CpuOracleBackend(load_orc()),
                                                   LocalComm(world), n, world, 100 + world)
    for r, a in got.items():
        assert np.max(np.abs(a - want[r << nl:(r + 1) << nl])) < 1e-12
    assert abs(e_got - e_want) < 1e-10
    assert swaps > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from dsv_cpu_backend import CpuOracleBackend
    from paper_2601_09951_b200.dsv import DistributedStateVector, TorchComm

    dist.init_process_group("gloo", rank=rank, world_size=world)
    want, got, nl, e_want, e_got, swaps = run_case(DistributedStateVector, CpuOracleBackend(load_orc()),
                                                   TorchComm(dist), n, world, 7)
    a = got[rank]
    q.put((rank, float(np.max(np.abs(a - want[rank << nl:(rank + 1) << nl]))), e_got, e_want, swaps))
    dist.barrier()
    dist.destroy_process_group()


def test_dsv_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, e_got, e_want, swaps in res:
        assert err < 1e-12
        assert abs(e_got - e_want) < 1e-10
        assert swaps > 0


@pytest.mark.parametrize("world,n", [(2, 7), (8, 9)])
def test_dsv_apply_circuit_runs(world, n):
    # apply_circuit: local runs go through the backend as one circuit (here
    # the CPU backend has no fused path: per-gate fallback), global-wire
    # gates through swaps; same amplitudes as the oracle
    from dsv_cpu_backend import CpuOracleBackend
    from paper_2601_09951_b200.dsv import DistributedStateVector, LocalComm

    orc = load_orc()
    pr = random.Random(300 + n)
    psi = random_state(np.random.default_rng(n), n)
    d = DistributedStateVector(n, world, CpuOracleBackend(orc), LocalComm(world))
    d.set_full(psi)
    gates = [(1, 0.1 * (q + 1), [q]) for q in range(n)] + [(2, 0.0, [q, q + 1]) for q in range(n - 1)]
    gates += circuit(pr, n, 20)
    d.apply_circuit(gates)
    want = orc.apply_gates(n, psi, gates)
    nl = n - (world.bit_length() - 1)
    for r, a in d.local_amplitudes().items():
        assert np.max(np.abs(a - want[r << nl:(r + 1) << nl])) < 1e-12
    assert d.swaps_done > 0
