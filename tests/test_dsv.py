"""Distributed state vector (BASELINE config 5) on CPU: the library's
planner (vqf_dsv_plan_circuit / vqf_dsv_plan_expectation, csrc/dsv.cu)
executed on numpy shards with the CPU oracle as the per-shard engine
(tests/dsv_numpy.py), against a single-state oracle run: amplitudes 1e-12,
energies 1e-10.  Virtual ranks (world 2/4/8) and world_size-2 gloo
processes; lazy layout (no swap back, Belady eviction); memory budget at
config-5 sizes."""
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

from oracle.oracle import Ham, load_orc, random_hamiltonian, random_state  # noqa: E402


def circuit(pr, n, count):
    gates = []
    for _ in range(count):
        k = pr.randint(0, 4)
        ws = pr.sample(range(n), [1, 1, 2, 4, 2][k])
        gates.append((k, pr.uniform(-3, 3), ws))
    # global wires (0..g-1) in every role
    gates += [(1, 0.7, [0]), (2, 0.0, [0, n - 1]), (2, 0.0, [n - 2, 1]), (3, 0.4, [1, 0, n - 1, 3]), (4, 0.9, [2, 0])]
    return gates


def hamiltonian(orc, pr, n):
    h = orc.canonicalize(random_hamiltonian(pr, n, 20))
    terms = list(h.terms)
    # strings with X/Y on every qubit: no I/Z local partner, cross-shard pairs
    terms.append((0.37, [(q, 1 + (q % 2)) for q in range(n)]))
    terms.append((-0.21, [(q, 1) for q in range(n)]))
    return Ham(n, terms)


@pytest.mark.parametrize("world,n", [(2, 7), (4, 8), (8, 9), (4, 10), (8, 11)])
def test_dsv_plans_match_single_state(world, n):
    from dsv_numpy import NumpyDsv

    orc = load_orc()
    pr = random.Random(1000 + 10 * world + n)
    psi = random_state(np.random.default_rng(n + world), n)
    d = NumpyDsv(orc, n, world, range(world))
    d.set_full(psi)
    gates = circuit(pr, n, 30)
    d.apply_circuit(gates)
    want = orc.apply_gates(n, psi, gates)
    assert np.max(np.abs(d.full() - want)) < 1e-12
    assert sorted(d.layout) == list(range(n))
    h = hamiltonian(orc, pr, n)
    assert abs(d.expectation(h) - orc.expectation(n, want, h)) < 1e-10
    # the layout the expectation left behind is a valid starting point
    more = circuit(pr, n, 10)
    d.apply_circuit(more)
    want = orc.apply_gates(n, want, more)
    assert np.max(np.abs(d.full() - want)) < 1e-12


def test_dsv_layout_is_lazy():
    """A hardware-efficient layer on 10 qubits over 8 ranks: every global
    qubit is swapped in once and never swapped back; the next layer reuses
    the layout (Belady eviction keeps soon-used qubits local)."""
    from paper_2601_09951_b200 import _capi as A
    from paper_2601_09951_b200 import dsv as D

    n, world = 10, 8
    layer = [(1, 0.1 * (q + 1), [q]) for q in range(n)] + [(2, 0.0, [q, q + 1]) for q in range(n - 1)]
    ops, mapped, layout = D.plan_circuit(n, world, list(range(n)), layer)
    swaps = [o for o in ops if o[0] == A.DSV_SWAP]
    # RYs on local wires run first; the 3 global qubits come in evicting
    # qubits whose RY is done; the CNOT chain brings 3 back: 6 exchanges
    assert len(swaps) <= 6
    assert sorted(layout) == list(range(n)) and layout != list(range(n))
    assert all(0 <= w < n - 3 for k, a, ws in mapped for w in ws)
    ops2, _, layout2 = D.plan_circuit(n, world, layout, layer)
    assert len([o for o in ops2 if o[0] == A.DSV_SWAP]) <= len(swaps) + 2
    # an eager swap-in / swap-back scheme pays two exchanges per global touch
    eager = 2 * sum(1 for k, a, ws in layer for w in ws if w < 3)
    assert len(swaps) < eager


def test_dsv_plan_errors():
    from paper_2601_09951_b200 import dsv as D

    with pytest.raises(ValueError, match="power of two"):
        D.plan_circuit(8, 3, list(range(8)), [(1, 0.1, [0])])
    with pytest.raises(ValueError, match="5 local qubits"):
        D.plan_circuit(6, 4, list(range(6)), [(1, 0.1, [0])])
    with pytest.raises(ValueError, match="permutation"):
        D.plan_circuit(8, 2, [0] * 8, [(1, 0.1, [0])])
    with pytest.raises(ValueError, match="wire"):
        D.plan_circuit(8, 2, list(range(8)), [(1, 0.1, [9])])


def test_dsv_memory_budget_config5():
    """Config 5: n = 35 fp64 over 8 GPUs = 64 GiB shards; per GPU the shard
    plus two 256 MiB exchange buffers (<= 1.5x a shard, < 180 GB); n = 34
    fp32 = 16 GiB shards; n = 36 fp64 still fits (128 GiB + 0.5 GiB)."""
    from paper_2601_09951_b200 import dsv as D

    gib = 1 << 30
    m35 = D.memory_per_gpu(35, 8, "f64")
    assert m35 == 64 * gib + 512 * (1 << 20)
    assert m35 <= 1.5 * 64 * gib
    assert D.memory_per_gpu(34, 8, "f32") == 16 * gib + 512 * (1 << 20)
    assert D.memory_per_gpu(36, 8, "f64") < 180e9
    assert D.memory_per_gpu(20, 4, "f64", chunk_bytes=1 << 20) == (1 << 18) * 16 + 2 * (1 << 20)
    assert D.memory_per_gpu(20, 4, "f64", one_shard_per_process=False) == (1 << 20) * 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, n, seed, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from dsv_numpy import NumpyDsv

    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = load_orc()
    pr = random.Random(seed)
    psi = random_state(np.random.default_rng(seed), n)
    d = NumpyDsv(orc, n, world, [rank], dist=dist)
    d.set_full(psi)
    gates = circuit(pr, n, 25)
    d.apply_circuit(gates)
    h = hamiltonian(orc, pr, n)
    e = d.expectation(h)
    out.put((rank, d.shards[rank], list(d.layout), e))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8)])
def test_dsv_gloo_processes_match_single_state(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seed = 4242
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    from paper_2601_09951_b200 import dsv as D

    orc = load_orc()
    pr = random.Random(seed)
    psi = random_state(np.random.default_rng(seed), n)
    gates = circuit(pr, n, 25)
    want = orc.apply_gates(n, psi, gates)
    h = hamiltonian(orc, pr, n)
    layout = res[0][2]
    assert all(r[2] == layout for r in res)
    got = D.to_logical(np.concatenate([r[1] for r in res]), layout)
    assert np.max(np.abs(got - want)) < 1e-12
    e_want = orc.expectation(n, want, h)
    assert all(abs(r[3] - e_want) < 1e-10 for r in res)
