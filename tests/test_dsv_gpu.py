"""Distributed state vector through the C ABI (vqf_dsv_*, csrc/dsv.cu) on
one B200: virtual ranks (every shard on the device, exchanges as in-place
device swaps) against the CPU oracle and the single-state engine, fp64 and
fp32; and two processes sharing the GPU, one shard each, exchanging through
the communicator callbacks (torch.distributed gloo staging through host
memory) in small chunks, so the chunked pack / sendrecv / unpack and the
chunked cross-shard expectation run for real."""
from __future__ import annotations

import os
import random
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle.oracle import Ham, random_hamiltonian, random_state

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gates_for(pr, n, count):
    out = []
    for _ in range(count):
        k = pr.randint(0, 4)
        ws = pr.sample(range(n), [1, 1, 2, 4, 2][k])
        out.append((k, pr.uniform(-3, 3), ws))
    out += [(1, 0.7, [0]), (2, 0.0, [0, n - 1]), (2, 0.0, [n - 2, 1]), (3, 0.4, [1, 0, n - 1, 3]), (4, 0.9, [2, 0])]
    return out


def hea_layer(n):
    return [(1, 0.1 * (q + 1), [q]) for q in range(n)] + [(2, 0.0, [q, q + 1]) for q in range(n - 1)]


def ham_with_cross(orc, pr, n, count=24):
    h = orc.canonicalize(random_hamiltonian(pr, n, count))
    terms = list(h.terms) + [(0.37, [(q, 1 + (q % 2)) for q in range(n)]), (-0.21, [(q, 1) for q in range(n)])]
    return Ham(n, terms)


@pytest.mark.parametrize("n,world", [(12, 4), (13, 8)])
def test_dsv_virtual_ranks_match_oracle(gpu, orc, n, world):
    from paper_2601_09951_b200.dsv import DistributedStateVector

    pr = random.Random(n * 7 + world)
    psi0 = random_state(np.random.default_rng(n), n)
    d = DistributedStateVector(n, world)
    d.set_full(psi0)
    gs = hea_layer(n) + gates_for(pr, n, 30)
    d.apply_circuit(gs)
    want = orc.apply_gates(n, psi0, gs)
    assert np.max(np.abs(d.full_amplitudes() - want)) < 1e-12
    h = ham_with_cross(orc, pr, n)
    assert abs(d.expectation(h) - orc.expectation(n, want, h)) < 1e-10
    tf = orc.build_tfim(n, 1.0, 1.0)
    assert abs(d.expectation(tf) - orc.expectation(n, want, tf)) < 1e-10
    st = d.stats()
    assert st["swaps"] > 0 and st["bytes_sent"] > 0
    # a second circuit starts from the layout the expectation left
    more = gates_for(pr, n, 10)
    d.apply_circuit(more)
    assert np.max(np.abs(d.full_amplitudes() - orc.apply_gates(n, want, more))) < 1e-12


@pytest.mark.parametrize("n,world,dtype", [(20, 8, "f64"), (18, 4, "f32")])
def test_dsv_virtual_ranks_match_engine(gpu, n, world, dtype):
    from paper_2601_09951_b200.dsv import DistributedStateVector

    V = gpu
    pr = random.Random(100 + n)
    psi0 = random_state(np.random.default_rng(n + 3), n)
    gs = hea_layer(n) + gates_for(pr, n, 40) + hea_layer(n)
    d = DistributedStateVector(n, world, dtype=dtype)
    d.set_full(psi0)
    d.apply_circuit(gs)
    single = V.StateVector(n)
    single.amplitudes = psi0
    V.apply_circuit(single, [V.Gate(k, a, tuple(w)) for k, a, w in gs])
    want = single.amplitudes
    tol_a, tol_e = (1e-12, 1e-10) if dtype == "f64" else (2e-6, 1e-5)
    assert np.max(np.abs(d.full_amplitudes() - want)) < tol_a
    tf = V.build_tfim(n, 1.0, 0.8)
    assert abs(d.expectation(tf) - V.expectation(single, tf)) < tol_e * max(1.0, n / 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _proc_worker(rank, world, port, n, seed, chunk, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from oracle.oracle import load_orc
    from paper_2601_09951_b200 import vqeforge as V
    from paper_2601_09951_b200.dsv import DistributedStateVector, TorchComm

    dist.init_process_group("gloo", rank=rank, world_size=world)
    V.init(0)
    orc = load_orc()
    pr = random.Random(seed)
    psi0 = random_state(np.random.default_rng(seed), n)
    d = DistributedStateVector(n, world, comm=TorchComm(dist, 0), chunk_bytes=chunk)
    d.set_full(psi0)
    gs = hea_layer(n) + gates_for(pr, n, 25)
    d.apply_circuit(gs)
    h = ham_with_cross(orc, pr, n)
    e = d.expectation(h)
    out.put((rank, d.shard(rank), d.layout(), e, d.stats()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,chunk", [(2, 12, 4096), (4, 12, 1 << 20)])
def test_dsv_processes_chunked_exchanges(gpu, orc, world, n, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seed = 77 + world
    procs = [ctx.Process(target=_proc_worker, args=(r, world, port, n, seed, chunk, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2601_09951_b200.dsv import to_logical

    pr = random.Random(seed)
    psi0 = random_state(np.random.default_rng(seed), n)
    gs = hea_layer(n) + gates_for(pr, n, 25)
    want = orc.apply_gates(n, psi0, gs)
    h = ham_with_cross(orc, pr, n)
    layout = res[0][2]
    assert all(r[2] == layout for r in res)
    got = to_logical(np.concatenate([r[1] for r in res]), layout)
    assert np.max(np.abs(got - want)) < 1e-12
    e_want = orc.expectation(n, want, h)
    assert all(abs(r[3] - e_want) < 1e-10 for r in res)
    assert all(r[4]["scratch_bytes"] >= 2 * min(chunk, (1 << (n - (world.bit_length() - 1))) * 16) for r in res)
