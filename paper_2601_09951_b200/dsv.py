"""Distributed state vector (BASELINE config 5: 34-35 qubits over 8 B200),
the Python face of the C ABI ``vqf_dsv_*`` (include/vqf_b200.h,
csrc/dsv.cu).

world = 2^g shards of 2^(n-g) amplitudes.  Qubits sit at positions
0..g-1 (global: position p is rank bit g-1-p) and g..n-1 (local: position p
is local index bit n-1-p, engine wire p-g of a shard).  The layout starts as
the identity and changes lazily: a gate or Pauli string that needs a global
qubit local swaps it with a local position (pairwise exchange of half a
shard with rank ^ (1 << bit)) and keeps the new layout.  Planning is done by
the library (``plan_circuit`` / ``plan_expectation`` expose it, host only).

Two placements:
  * virtual ranks (``comm=None``): every shard on one device, exchanges are
    in-place device swaps -- validates the distributed path on one GPU;
  * one shard per process (``comm=TorchComm(dist, device)``): exchanges in
    ``chunk_bytes`` pieces through two preallocated device buffers over
    torch.distributed point-to-point (NCCL over NVLink on B200; gloo stages
    through host memory), the expectation's totals through all_reduce.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as A
from . import vqeforge as V

GateLike = Tuple[int, float, Sequence[int]]


def _gates(gates) -> "C.Array":
    out = []
    for g in gates:
        if isinstance(g, V.Gate):
            out.append((g.kind, g.angle, g.wires))
        else:
            k, a, w = g
            out.append((k, a, tuple(w)))
    arr = (A.Gate * max(1, len(out)))()
    for i, (k, a, w) in enumerate(out):
        arr[i].kind = k
        arr[i].angle = a
        arr[i].n_wires = len(w)
        for j, q in enumerate(w):
            arr[i].wires[j] = q
    return arr, len(out)


def _ham(n: int, terms):
    """A QubitHamiltonian, or any (coefficient, [(qubit, axis)]) sequence /
    object with such .terms (term order is kept: plans index into it)."""
    if isinstance(terms, V.QubitHamiltonian):
        return terms
    terms = getattr(terms, "terms", terms)
    return V.QubitHamiltonian(n, [V.PauliTerm(c, list(a)) for c, a in terms])


def plan_circuit(n: int, world: int, layout: Sequence[int], gates) -> Tuple[list, list, List[int]]:
    """Host-only circuit plan: (ops, mapped gates, new layout).  ops are
    (kind, a, b, first, count) with kind A.DSV_SWAP / A.DSV_LOCAL."""
    arr, ng = _gates(gates)
    pos = (C.c_uint32 * n)(*layout)
    cap = 4 * ng + 8
    ops = (A.DsvOp * cap)()
    mapped = (A.Gate * max(1, ng))()
    nops = C.c_uint32()
    V.check(A.lib.vqf_dsv_plan_circuit(n, world, pos, arr, ng, ops, cap, C.byref(nops), mapped))
    o = [(ops[i].kind, ops[i].a, ops[i].b, ops[i].first, ops[i].count) for i in range(nops.value)]
    m = [(mapped[i].kind, mapped[i].angle, [mapped[i].wires[j] for j in range(mapped[i].n_wires)]) for i in range(ng)]
    return o, m, list(pos)


def plan_expectation(n: int, world: int, layout: Sequence[int], terms) -> Tuple[list, list, List[int]]:
    """Host-only expectation plan: (ops, planned terms, new layout).  A
    planned term is a dict of the vqf_dsv_term fields."""
    h = _ham(n, terms)
    keep, hs = h.as_c()
    pos = (C.c_uint32 * n)(*layout)
    cap = 4 * len(h.terms) + 8
    ops = (A.DsvOp * cap)()
    pts = (A.DsvTerm * max(1, len(h.terms)))()
    nops = C.c_uint32()
    V.check(A.lib.vqf_dsv_plan_expectation(n, world, pos, C.byref(hs), ops, cap, C.byref(nops), pts))
    o = [(ops[i].kind, ops[i].a, ops[i].b, ops[i].first, ops[i].count) for i in range(nops.value)]
    fields = [f for f, _ in A.DsvTerm._fields_ if f != "pad"]
    t = [{f: int(getattr(pts[i], f)) for f in fields} for i in range(len(h.terms))]
    return o, t, list(pos)


def memory_per_gpu(n: int, world: int, dtype: str = "f64", chunk_bytes: int = 0, one_shard_per_process: bool = True) -> int:
    return int(A.lib.vqf_dsv_memory_per_gpu(n, world, A.F64 if dtype == "f64" else A.F32, chunk_bytes,
                                            1 if one_shard_per_process else 0))


class TorchComm:
    """torch.distributed point-to-point for the library's exchanges: one
    shard per process.  NCCL exchanges device memory directly; gloo (CPU
    tests, several processes sharing one GPU) stages through host memory."""

    def __init__(self, dist, device: int = 0):
        import torch

        self.torch = torch
        self.dist = dist
        self.rank = dist.get_rank()
        self.device = device
        self.nccl = dist.get_backend() == "nccl"
        self._sr = A.SENDRECV_FN(self._sendrecv)
        self._ar = A.ALLREDUCE_FN(self._allreduce)

    def _dev_bytes(self, ptr: int, nbytes: int):
        class _Cai:
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
                                        "strides": None}

        return self.torch.as_tensor(_Cai(), device=f"cuda:{self.device}")

    def _sendrecv(self, user, send_ptr, recv_ptr, nbytes, peer, stream):
        try:
            torch = self.torch
            torch.cuda.ExternalStream(stream, device=self.device).synchronize() if stream else torch.cuda.synchronize()
            send = self._dev_bytes(send_ptr, nbytes)
            recv = self._dev_bytes(recv_ptr, nbytes)
            if self.nccl:
                reqs = self.dist.batch_isend_irecv([self.dist.P2POp(self.dist.isend, send, int(peer)),
                                                    self.dist.P2POp(self.dist.irecv, recv, int(peer))])
                for r in reqs:
                    r.wait()
                torch.cuda.synchronize(self.device)
            else:
                hs = send.cpu()
                hr = torch.empty_like(hs)
                reqs = [self.dist.isend(hs, int(peer)), self.dist.irecv(hr, int(peer))]
                for r in reqs:
                    r.wait()
                recv.copy_(hr)
                torch.cuda.synchronize(self.device)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed exchange
            return 1

    def _allreduce(self, user, values, count):
        try:
            t = self.torch.tensor([values[i] for i in range(count)], dtype=self.torch.float64,
                                  device=f"cuda:{self.device}" if self.nccl else "cpu")
            self.dist.all_reduce(t)
            for i in range(count):
                values[i] = float(t[i])
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def as_c(self) -> A.DsvComm:
        return A.DsvComm(self.rank, self._sr, self._ar, None)


class DistributedStateVector:
    """An n-qubit state over `world` shards (see module doc)."""

    def __init__(self, n: int, world: int, dtype: str = "f64", device: int = 0, comm: Optional[TorchComm] = None,
                 chunk_bytes: int = 0):
        self.n, self.world, self.dtype, self.device = n, world, dtype, device
        self.g = world.bit_length() - 1
        self.nl = n - self.g
        self.comm = comm
        self._c = comm.as_c() if comm is not None else None
        self._h = A.DSV()
        V.check(A.lib.vqf_dsv_create(n, world, A.F64 if dtype == "f64" else A.F32, device,
                                     C.byref(self._c) if self._c is not None else None, chunk_bytes,
                                     C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            A.lib.vqf_dsv_destroy(h)
            self._h = A.DSV()

    @property
    def ranks(self) -> List[int]:
        return [self.comm.rank] if self.comm is not None else list(range(self.world))

    def apply_circuit(self, gates) -> None:
        arr, ng = _gates(gates)
        V.check(A.lib.vqf_dsv_apply_circuit(self._h, arr, ng))

    def apply_gate(self, kind: int, angle: float, wires: Sequence[int]) -> None:
        self.apply_circuit([(kind, angle, wires)])

    def expectation(self, terms) -> float:
        h = _ham(self.n, terms)
        keep, hs = h.as_c()
        out = np.zeros(1)
        V.check(A.lib.vqf_dsv_expectation(self._h, C.byref(hs), out.ctypes.data_as(A.dp)))
        return float(out[0])

    def layout(self) -> List[int]:
        pos = (C.c_uint32 * self.n)()
        V.check(A.lib.vqf_dsv_layout(self._h, pos))
        return list(pos)

    def stats(self) -> dict:
        s, b, m = C.c_uint64(), C.c_uint64(), C.c_uint64()
        V.check(A.lib.vqf_dsv_stats(self._h, C.byref(s), C.byref(b), C.byref(m)))
        return {"swaps": s.value, "bytes_sent": b.value, "scratch_bytes": m.value}

    def shard(self, rank: int) -> np.ndarray:
        out = np.zeros(2 << self.nl)
        V.check(A.lib.vqf_dsv_shard_download(self._h, rank, out.ctypes.data_as(A.dp)))
        return out.view(np.complex128)

    def set_shard(self, rank: int, amps: np.ndarray) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128).view(np.float64)
        V.check(A.lib.vqf_dsv_shard_upload(self._h, rank, a.ctypes.data_as(A.dp)))

    # logical <-> physical order (virtual ranks hold every shard)
    def full_amplitudes(self) -> np.ndarray:
        phys = np.concatenate([self.shard(r) for r in range(self.world)])
        return to_logical(phys, self.layout())

    def set_full(self, amps: np.ndarray) -> None:
        phys = to_physical(np.asarray(amps, dtype=np.complex128), self.layout())
        for r in self.ranks:
            self.set_shard(r, phys[r << self.nl:(r + 1) << self.nl])


def to_logical(phys: np.ndarray, layout: Sequence[int]) -> np.ndarray:
    """Physical axis a of the 2^n tensor is position a (MSB first); logical
    axis q is the qubit at layout[q]."""
    n = len(layout)
    return np.ascontiguousarray(phys.reshape([2] * n).transpose(list(layout))).reshape(-1)


def to_physical(logical: np.ndarray, layout: Sequence[int]) -> np.ndarray:
    n = len(layout)
    inv = [0] * n
    for q, p in enumerate(layout):
        inv[p] = q
    return np.ascontiguousarray(logical.reshape([2] * n).transpose(inv)).reshape(-1)
