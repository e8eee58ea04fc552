"""Distributed state vector (BASELINE config 5: 34-35 qubits over 8 B200).

Layout (MSB-first, statevector.hpp:30-31): with world = 2^g ranks, wires
0..g-1 are *global* — they select the rank (rank r holds the amplitudes whose
top g index bits equal r); wires g..n-1 are local wires 0..n-g-1 of every
shard.  Each shard is an ordinary engine state (vqf_sv, HBM-resident).

* A gate on local wires runs the engine's kernel on every shard.
* A gate touching global wire w first swaps w with a free local wire t (the
  highest local wire not used by the gate): rank r exchanges the half of its
  shard whose bit t differs from its own bit for w with rank r ^ (1 << (g-1-w))
  — one contiguous block when t is the top local wire — then the gate runs
  locally on t, then the swap is undone (it is an involution).
* Expectation: terms without X/Y on global wires are local (a Z on a global
  wire is a sign fixed by the rank's bits); terms flipping global wires are
  grouped by their global flip set, those wires swapped into local positions
  outside the group's support, evaluated, swapped back.  Shard partials are
  all-reduced (two doubles) and the imaginary-residue check of
  statevector.hpp:244-247 applies to the total.

Exchanges are delegated to a communicator: direct device copies between
shards living in this process (virtual ranks, used to validate the path on
one GPU) and torch.distributed send/recv (NCCL over NVLink) between
processes.  The local compute is a backend: `GpuBackend` (the engine, via the
C ABI) in the product; tests plug a CPU backend.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

AXIS_X, AXIS_Y, AXIS_Z = 1, 2, 3


def half_blocks(nl: int, b: int, v: int) -> List[Tuple[int, int]]:
    """(start, length) runs of local indices whose bit b equals v."""
    step = 1 << (b + 1)
    return [(j * step + (v << b), 1 << b) for j in range(1 << (nl - 1 - b))]


class GpuBackend:
    """Shards as engine states on one CUDA device."""

    def __init__(self, device: int = 0):
        from . import vqeforge as V

        self.V = V
        self.device = device

    def zero_state(self, nl: int, holds_origin: bool):
        psi = self.V.StateVector(nl, device=self.device)  # |0..0> of the shard
        if not holds_origin:
            psi.amplitudes = np.zeros(1 << nl, dtype=np.complex128)
        return psi

    def set_amplitudes(self, psi, amps: np.ndarray) -> None:
        psi.amplitudes = amps

    def amplitudes(self, psi) -> np.ndarray:
        return psi.amplitudes

    def view(self, psi):
        """The shard as a torch float64 tensor [2^nl, 2] aliasing HBM."""
        import torch

        ptr, nbytes = C.c_void_p(), C.c_uint64()
        self.V.check(self.V.lib.vqf_sv_device_ptr(psi._h, C.byref(ptr), C.byref(nbytes)))

        class _Cai:
            __cuda_array_interface__ = {"shape": (nbytes.value // 16, 2), "typestr": "<f8",
                                        "data": (ptr.value, False), "version": 3, "strides": None}

        return torch.as_tensor(_Cai(), device=f"cuda:{self.device}")

    def apply(self, psi, kind: int, angle: float, wires: Sequence[int]) -> None:
        self.V.apply_gate(psi, self.V.Gate(kind, angle, tuple(wires)))

    def apply_circuit(self, psi, gates) -> None:
        """A run of local gates as fused tile passes (vqf_apply_circuit)."""
        self.V.apply_circuit(psi, [self.V.Gate(k, a, tuple(w)) for k, a, w in gates])

    def expectation_complex(self, psi, nl: int, terms) -> complex:
        if not terms:
            return 0j
        h = self.V.QubitHamiltonian(nl, [self.V.PauliTerm(c, a) for c, a in terms])
        keep, hs = h.as_c()
        out = np.zeros(2)
        self.V.check(self.V.lib.vqf_expectation_complex(psi._h, C.byref(hs), out.ctypes.data_as(self.V.A.dp)))
        return complex(out[0], out[1])

    def temp_state(self, nl: int):
        return self.V.StateVector(nl, device=self.device)

    def cross_expectation(self, a, b, nl: int, terms) -> complex:
        h = self.V.QubitHamiltonian(nl, [self.V.PauliTerm(c, ax) for c, ax in terms])
        keep, hs = h.as_c()
        out = np.zeros(2)
        self.V.check(self.V.lib.vqf_cross_expectation(a._h, b._h, C.byref(hs), out.ctypes.data_as(self.V.A.dp)))
        return complex(out[0], out[1])


class LocalComm:
    """Every rank lives in this process (virtual ranks on one device)."""

    def __init__(self, world: int):
        self.world = world

    def local_ranks(self, world: int) -> List[int]:
        return list(range(world))

    def allreduce(self, value: complex) -> complex:
        return value  # the caller already summed every shard

    def fetch(self, src: Dict[int, object], dst: Dict[int, object], peer_of) -> None:
        for r, d in dst.items():
            d.copy_(src[peer_of(r)])

    def exchange(self, views: Dict[int, object], blocks_of, peer_of) -> None:
        done = set()
        for r, v in views.items():
            p = peer_of(r)
            if (min(r, p), max(r, p)) in done:
                continue
            done.add((min(r, p), max(r, p)))
            vp = views[p]
            for (sr, ln), (sp, _) in zip(blocks_of(r), blocks_of(p)):
                tmp = v[sr:sr + ln].clone()
                v[sr:sr + ln].copy_(vp[sp:sp + ln])
                vp[sp:sp + ln].copy_(tmp)


class TorchComm:
    """One rank per process; exchanges with torch.distributed P2P (NCCL over
    NVLink on B200, gloo in CPU tests)."""

    def __init__(self, dist, device: Optional[str] = None):
        self.dist = dist
        self.rank = dist.get_rank()
        self.device = device

    def local_ranks(self, world: int) -> List[int]:
        return [self.rank]

    def allreduce(self, value: complex) -> complex:
        import torch

        t = torch.tensor([value.real, value.imag], dtype=torch.float64, device=self.device or "cpu")
        self.dist.all_reduce(t)
        return complex(float(t[0]), float(t[1]))

    def fetch(self, src: Dict[int, object], dst: Dict[int, object], peer_of) -> None:
        (r, v), = src.items()
        p = peer_of(r)
        send = v.clone()
        ops = [self.dist.P2POp(self.dist.isend, send, p), self.dist.P2POp(self.dist.irecv, dst[r], p)]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()

    def exchange(self, views: Dict[int, object], blocks_of, peer_of) -> None:
        (r, v), = views.items()
        p = peer_of(r)
        ops, recvs = [], []
        for (sr, ln), _ in zip(blocks_of(r), blocks_of(p)):
            send = v[sr:sr + ln].clone()
            recv = v[sr:sr + ln]
            ops.append(self.dist.P2POp(self.dist.isend, send, p))
            buf = recv.clone() if not recv.is_contiguous() else recv
            ops.append(self.dist.P2POp(self.dist.irecv, buf, p))
            recvs.append((recv, buf, send))
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()
        for recv, buf, _ in recvs:
            if buf is not recv:
                recv.copy_(buf)


class DistributedStateVector:
    """An n-qubit state split over `world` = 2^g shards (see module doc)."""

    def __init__(self, n: int, world: int, backend, comm):
        g = world.bit_length() - 1
        if (1 << g) != world:
            raise ValueError("world size must be a power of two")
        if n - g < 5:
            raise ValueError("need at least 5 local qubits per shard")
        self.n, self.world, self.g, self.nl = n, world, g, n - g
        self.backend, self.comm = backend, comm
        self.shards = {r: backend.zero_state(self.nl, r == 0) for r in comm.local_ranks(world)}
        self.swaps_done = 0

    # ------------------------------------------------------------ layout
    def rank_bit(self, rank: int, w: int) -> int:
        return (rank >> (self.g - 1 - w)) & 1

    def swap(self, w: int, t: int) -> None:
        """Exchanges global wire w with local wire t (t >= g) on every rank."""
        p = self.g - 1 - w
        b = self.nl - 1 - (t - self.g)  # t's bit in the local index
        views = {r: self.backend.view(s) for r, s in self.shards.items()}
        self.comm.exchange(views, lambda r: half_blocks(self.nl, b, 1 - ((r >> p) & 1)), lambda r: r ^ (1 << p))
        self.swaps_done += 1

    def _free_local(self, taken: Iterable[int], count: int) -> List[int]:
        taken = set(taken)
        out = []
        for t in range(self.g, self.n):  # top local wire first: one contiguous block
            if t not in taken:
                out.append(t)
                taken.add(t)
                if len(out) == count:
                    return out
        raise ValueError("not enough free local wires for the swap")

    # ------------------------------------------------------------- gates
    def apply_gate(self, kind: int, angle: float, wires: Sequence[int]) -> None:
        glob = [w for w in wires if w < self.g]
        partners = self._free_local(wires, len(glob)) if glob else []
        for w, t in zip(glob, partners):
            self.swap(w, t)
        remap = dict(zip(glob, partners))
        local = [remap.get(w, w) - self.g for w in wires]
        for s in self.shards.values():
            self.backend.apply(s, kind, angle, local)
        for w, t in reversed(list(zip(glob, partners))):
            self.swap(w, t)

    def apply_circuit(self, gates: Sequence[Tuple[int, float, Sequence[int]]]) -> None:
        """apply_circuit (statevector.hpp:205-207) on the sharded state: maximal
        runs of gates on local wires go to the backend as one fused circuit
        per shard (tile passes); a gate touching a global wire is swapped in,
        applied and swapped back (apply_gate)."""
        fused = getattr(self.backend, "apply_circuit", None)
        run: List[Tuple[int, float, List[int]]] = []

        def flush():
            if not run:
                return
            for sh in self.shards.values():
                if fused is not None:
                    fused(sh, run)
                else:
                    for k, a, w in run:
                        self.backend.apply(sh, k, a, w)
            run.clear()

        for kind, angle, wires in gates:
            if all(w >= self.g for w in wires):
                run.append((kind, angle, [w - self.g for w in wires]))
            else:
                flush()
                self.apply_gate(kind, angle, wires)
        flush()

    # ------------------------------------------------------- expectation
    def _partition(self, ts, f):
        """Splits a group with global flip set f into subgroups that share
        len(f) swap partners: local wires on which every term of the
        subgroup acts as I or Z (after the swap that operator sits on the
        global wire, where I is nothing and Z is this rank's sign)."""
        out = []
        rest = list(ts)
        while rest:
            ok = [t for t in range(self.g, self.n)]
            sub = []
            for term in list(rest):
                axes = dict(term[1])
                cand = [t for t in ok if axes.get(t, 0) in (0, AXIS_Z)]
                if len(cand) >= len(f):
                    ok = cand
                    sub.append(term)
                    rest.remove(term)
            if not sub:  # flips f and X/Y on every local wire: cross-shard terms
                return out, rest
            # prefer the top local wires: one contiguous exchange block
            out.append((sub, ok[:len(f)]))
        return out, []

    def expectation(self, terms: Sequence[Tuple[complex, Sequence[Tuple[int, int]]]]) -> float:
        """terms: [(coefficient, [(wire, axis)])] as PauliTerm (pauli.hpp:65)."""
        groups: Dict[Tuple[int, ...], list] = {}
        for c, axes in terms:
            f = tuple(sorted(q for q, a in axes if q < self.g and a in (AXIS_X, AXIS_Y)))
            groups.setdefault(f, []).append((c, list(axes)))
        total = 0j
        for f, ts in groups.items():
            subgroups, leftover = self._partition(ts, f) if f else ([(ts, [])], [])
            if leftover:
                total += self._cross_terms(f, leftover)
            for sub, partners in subgroups:
                for w, t in zip(f, partners):
                    self.swap(w, t)
                # after the swaps, qubit w lives on local wire t and qubit t on global wire w
                loc = dict(zip(f, partners))
                glob = {t: w for w, t in loc.items()}
                for r, s in self.shards.items():
                    local_terms = []
                    for c, axes in sub:
                        coeff = complex(c)
                        ax = []
                        for q, a in axes:
                            if q in loc:
                                ax.append((loc[q] - self.g, a))
                            elif q in glob:  # I/Z by construction: Z is the sign of global wire glob[q]
                                if a == AXIS_Z and self.rank_bit(r, glob[q]):
                                    coeff = -coeff
                            elif q < self.g:  # Z on an untouched global wire
                                if self.rank_bit(r, q):
                                    coeff = -coeff
                            else:
                                ax.append((q - self.g, a))
                        local_terms.append((coeff, sorted(ax)))
                    total += self.backend.expectation_complex(s, self.nl, local_terms)
                for w, t in reversed(list(zip(f, partners))):
                    self.swap(w, t)
        total = self.comm.allreduce(total)
        if abs(total.imag) >= 1e-10:  # statevector.hpp:244-247
            raise RuntimeError("expectation has imaginary residue %f" % total.imag)
        return total.real

    def _cross_terms(self, f, terms) -> complex:
        """Terms flipping global wires f (rank mask M) and no swappable local
        wire: every rank r fetches shard r ^ M and evaluates
        sum_l conj(psi_r[l]) (-1)^popc(l & yz_l) psi_{r^M}[l ^ flip_l] with the
        global part of the phase folded into the coefficient."""
        M = 0
        for w in f:
            M |= 1 << (self.g - 1 - w)
        views = {r: self.backend.view(s) for r, s in self.shards.items()}
        tmp = {r: self.backend.temp_state(self.nl) for r in self.shards}
        self.comm.fetch(views, {r: self.backend.view(t) for r, t in tmp.items()}, lambda r: r ^ M)
        total = 0j
        for r, s in self.shards.items():
            local_terms = []
            for c, axes in terms:
                coeff = complex(c)
                ax = []
                for q, a in axes:
                    if q < self.g:
                        bit = self.rank_bit(r, q)
                        if a == AXIS_Y:
                            coeff *= -1j  # (-i) per Y
                        if a in (AXIS_Y, AXIS_Z) and bit:
                            coeff = -coeff
                    else:
                        ax.append((q - self.g, a))
                local_terms.append((coeff, sorted(ax)))
            total += self.backend.cross_expectation(s, tmp[r], self.nl, local_terms)
        self.swaps_done += 1
        return total

    # ----------------------------------------------------------- testing
    def set_full(self, amps: np.ndarray) -> None:
        """Scatters a full 2^n state (tests)."""
        amps = np.asarray(amps, dtype=np.complex128).reshape(self.world, 1 << self.nl)
        for r, s in self.shards.items():
            self.backend.set_amplitudes(s, amps[r])

    def local_amplitudes(self) -> Dict[int, np.ndarray]:
        return {r: self.backend.amplitudes(s) for r, s in self.shards.items()}
