"""TEST INFRASTRUCTURE: executes the library's distributed plans
(vqf_dsv_plan_circuit / vqf_dsv_plan_expectation, csrc/dsv.cu) on numpy
shards with the CPU oracle as the per-shard engine, so the planner -- layout,
lazy swaps, term folding, cross-shard pairs -- is checked on CPU against a
single-state oracle run.  Ranks are virtual (all shards here) or one per
process (exchanges over torch.distributed gloo)."""
from __future__ import annotations

import numpy as np

from paper_2601_09951_b200 import _capi as A
from paper_2601_09951_b200 import dsv as D

MI = [1, -1j, -1, 1j]  # (-i)^k


def put_bit(k: np.ndarray, b: int, v: int) -> np.ndarray:
    low = k & ((1 << b) - 1)
    return ((k >> b) << (b + 1)) | (v << b) | low


def half_index(nl: int, b: int, v: int) -> np.ndarray:
    return put_bit(np.arange(1 << (nl - 1), dtype=np.int64), b, v)


def popc_parity(x: np.ndarray) -> np.ndarray:
    x = x.copy()
    p = np.zeros_like(x)
    while np.any(x):
        p ^= x & 1
        x >>= 1
    return p


class NumpyDsv:
    def __init__(self, orc, n: int, world: int, ranks, dist=None):
        self.orc, self.n, self.world = orc, n, world
        self.g = world.bit_length() - 1
        self.nl = n - self.g
        self.layout = list(range(n))
        self.dist = dist
        self.shards = {r: np.zeros(1 << self.nl, dtype=np.complex128) for r in ranks}
        if 0 in self.shards:
            self.shards[0][0] = 1.0
        self.swaps = 0

    def set_full(self, amps):
        phys = D.to_physical(np.asarray(amps, dtype=np.complex128), self.layout)
        for r in self.shards:
            self.shards[r] = phys[r << self.nl:(r + 1) << self.nl].copy()

    def full(self):
        phys = np.concatenate([self.shards[r] for r in range(self.world)])
        return D.to_logical(phys, self.layout)

    # ------------------------------------------------------------- ops
    def _exchange(self, r, send: np.ndarray) -> np.ndarray:
        import torch

        peer = self._peer
        s = torch.from_numpy(np.ascontiguousarray(send).view(np.float64))
        rcv = torch.empty_like(s)
        reqs = [self.dist.isend(s, peer), self.dist.irecv(rcv, peer)]
        for q in reqs:
            q.wait()
        return rcv.numpy().view(np.complex128)

    def swap(self, pg: int, pl: int):
        rb, b = self.g - 1 - pg, self.n - 1 - pl
        if self.dist is None:
            for r in range(self.world):
                p = r ^ (1 << rb)
                if p < r:
                    continue
                ir = half_index(self.nl, b, 1 - ((r >> rb) & 1))
                ip = half_index(self.nl, b, 1 - ((p >> rb) & 1))
                tmp = self.shards[r][ir].copy()
                self.shards[r][ir] = self.shards[p][ip]
                self.shards[p][ip] = tmp
        else:
            (r,) = self.shards
            self._peer = r ^ (1 << rb)
            ir = half_index(self.nl, b, 1 - ((r >> rb) & 1))
            self.shards[r][ir] = self._exchange(r, self.shards[r][ir])
        pos = self.layout
        qa, qb = pos.index(pg), pos.index(pl)
        pos[qa], pos[qb] = pl, pg
        self.swaps += 1

    def apply_circuit(self, gates):
        ops, mapped, new = D.plan_circuit(self.n, self.world, self.layout, gates)
        for kind, a, b, first, count in ops:
            if kind == A.DSV_SWAP:
                self.swap(a, b)
            else:
                for r in self.shards:
                    self.shards[r] = self.orc.apply_gates(self.nl, self.shards[r], mapped[first:first + count])
        assert self.layout == new

    def _sum(self, h, pts, r, a: np.ndarray, b: np.ndarray) -> complex:
        l = np.arange(1 << self.nl, dtype=np.int64)
        tot = 0j
        for pt in pts:
            t = h.terms[pt["term"]]
            c = complex(t[0] if isinstance(t, tuple) else t.coefficient) * MI[(pt["l_ny"] + pt["g_ny"]) % 4]
            if bin(r & pt["g_yz"]).count("1") & 1:
                c = -c
            sign = 1 - 2 * popc_parity(l & pt["l_yz"])
            tot += c * np.sum(np.conj(a) * sign * b[l ^ pt["l_flip"]])
        return tot

    def expectation(self, h) -> float:
        ops, pts, new = D.plan_expectation(self.n, self.world, self.layout, h)
        tot = 0j
        for kind, a, b, first, count in ops:
            sel = pts[first:first + count]
            if kind == A.DSV_SWAP:
                self.swap(a, b)
            elif kind == A.DSV_EVAL:
                for r, s in self.shards.items():
                    tot += self._sum(h, sel, r, s, s)
            else:  # CROSS: rank r pairs with r ^ a
                for r, s in self.shards.items():
                    if self.dist is None:
                        other = self.shards[r ^ a]
                    else:
                        self._peer = r ^ a
                        other = self._exchange(r, s)
                    tot += self._sum(h, sel, r, s, other)
        assert self.layout == new
        if self.dist is not None:
            import torch

            t = torch.tensor([tot.real, tot.imag], dtype=torch.float64)
            self.dist.all_reduce(t)
            tot = complex(float(t[0]), float(t[1]))
        if abs(tot.imag) >= 1e-10:
            raise RuntimeError("expectation has imaginary residue %f" % tot.imag)
        return tot.real
