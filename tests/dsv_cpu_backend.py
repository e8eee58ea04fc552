"""TEST INFRASTRUCTURE: a CPU backend for paper_2601_09951_b200.dsv whose
local compute is the oracle (oracle/vqf_oracle.c) — so the distributed
orchestration (global-qubit swaps, sign handling, grouping, all-reduce) can
be checked on CPU against a single-state oracle run."""
from __future__ import annotations

import numpy as np
import torch


class CpuOracleBackend:
    def __init__(self, orc):
        self.orc = orc

    def zero_state(self, nl, holds_origin):
        a = np.zeros(1 << nl, dtype=np.complex128)
        if holds_origin:
            a[0] = 1.0
        return a

    def set_amplitudes(self, psi, amps):
        psi[:] = amps

    def amplitudes(self, psi):
        return psi.copy()

    def view(self, psi):
        return torch.from_numpy(psi.view(np.float64).reshape(-1, 2))

    def apply(self, psi, kind, angle, wires):
        nl = psi.size.bit_length() - 1
        psi[:] = self.orc.apply_gates(nl, psi, [(kind, angle, list(wires))])

    def temp_state(self, nl):
        return np.zeros(1 << nl, dtype=np.complex128)

    def cross_expectation(self, a, b, nl, terms):
        idx = np.arange(1 << nl, dtype=np.int64)
        total = 0j
        for c, axes in terms:
            flip = yz = 0
            ny = 0
            for q, ax in axes:
                bit = 1 << (nl - 1 - q)
                if ax in (1, 2):
                    flip |= bit
                if ax in (2, 3):
                    yz |= bit
                if ax == 2:
                    ny += 1
            sign = 1 - 2 * (np.bitwise_count(idx & yz) & 1).astype(np.int64)
            total += c * (-1j) ** ny * np.sum(sign * np.conj(a) * b[idx ^ flip])
        return complex(total)

    def expectation_complex(self, psi, nl, terms):
        # sum_t c_t (-i)^{n_y} sum_i (-1)^popc(i & yz) conj(psi_i) psi_{i ^ flip}
        idx = np.arange(1 << nl, dtype=np.int64)
        total = 0j
        for c, axes in terms:
            flip = yz = 0
            ny = 0
            for q, a in axes:
                bit = 1 << (nl - 1 - q)
                if a in (1, 2):
                    flip |= bit
                if a in (2, 3):
                    yz |= bit
                if a == 2:
                    ny += 1
            base = (-1j) ** ny
            sign = 1 - 2 * (np.bitwise_count(idx & yz) & 1).astype(np.int64)
            total += c * base * np.sum(sign * np.conj(psi) * psi[idx ^ flip])
        return complex(total)
