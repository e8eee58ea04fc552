"""Test helpers shared by the GPU parity tests."""
from __future__ import annotations


def ham_from_text(V, n_qubits, text):
    """Parses pauli.hpp:294 text into the product's QubitHamiltonian."""
    from oracle.oracle import Ham

    h = Ham.from_text(n_qubits, text)
    return V.QubitHamiltonian(n_qubits, [V.PauliTerm(c, axes) for c, axes in h.terms]), h
