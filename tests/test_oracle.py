"""CPU: pins the oracle restatement (oracle/vqf_oracle.c) against the
reference's own golden vectors and against the compiled reference
(oracle/_ref).  Citations are to /root/reference/proj/tests."""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

from oracle.oracle import Ham, random_hamiltonian, random_state

# test_chem.cpp:223-239 — frozen 15-term H2 Hamiltonian at 0.7414 A
GOLDEN_H2 = {
    "": -0.098863900993594683,
    "X0X1Y2Y3": -0.045322201306261987,
    "X0Y1Y2X3": 0.045322201306261987,
    "Y0X1X2Y3": 0.045322201306261987,
    "Y0Y1X2X3": -0.045322201306261987,
    "Z0": 0.17119775722238972,
    "Z0Z1": 0.16862219413401999,
    "Z0Z2": 0.1205448251164476,
    "Z0Z3": 0.16586702642270956,
    "Z1": 0.17119775722238978,
    "Z1Z2": 0.16586702642270956,
    "Z1Z3": 0.1205448251164476,
    "Z2": -0.22278595496571194,
    "Z2Z3": 0.17434844430984958,
    "Z3": -0.22278595496571194,
}


def test_h2_golden_hamiltonian(orc):
    h = orc.build_h2_hamiltonian(0.7414)
    assert len(h.terms) == 15
    for t in range(15):
        assert h.terms[t][0].imag == 0.0
        assert abs(h.terms[t][0].real - GOLDEN_H2[h.key(t)]) < 1e-12


def test_hf_golden(orc):
    # test_chem.cpp:139 HF energy at 1.4 bohr
    assert abs(orc.hartree_fock(1.4 / 1.8897259886)["hf_energy"] - (-1.1167143250625697)) < 1e-12


def test_exact_ground_energy_golden(ref):
    # test_chem.cpp:262-270
    assert abs(ref.exact_ground_energy(ref.build_h2_hamiltonian(0.7414)) - (-1.1372701752425913)) < 1e-9


def test_basis_and_gate_goldens(orc):
    # test_statevector.cpp:65-81
    a = orc.basis_state(4, [1, 1, 0, 0])
    assert a[12] == 1 and np.count_nonzero(a) == 1
    assert orc.basis_state(2, [0, 1])[1] == 1
    with pytest.raises(ValueError):
        orc.basis_state(2, [0, 1, 0])
    # test_statevector.cpp:116-132 DE(pi) and DE(0.6)
    out = orc.apply_gates(4, a, [(3, math.pi, [0, 1, 2, 3])])
    assert abs(out[3].real - 1.0) < 1e-15 and abs(out[12]) < 1e-15
    out = orc.apply_gates(4, a, [(3, 0.6, [0, 1, 2, 3])])
    assert abs(out[12].real - math.cos(0.3)) < 1e-15 and abs(out[3].real - math.sin(0.3)) < 1e-15
    b = orc.basis_state(4, [0, 1, 0, 1])
    assert np.array_equal(orc.apply_gates(4, b, [(3, 1.2, [0, 1, 2, 3])]), b)
    # test_statevector.cpp:96-114
    z = np.zeros(2, complex)
    z[0] = 1
    assert orc.apply_gates(1, z, [(0, 0.0, [0])])[1] == 1
    ry = orc.apply_gates(1, z, [(1, 1.0, [0])])
    assert abs(ry[0].real - math.cos(0.5)) < 1e-15 and abs(ry[1].real - math.sin(0.5)) < 1e-15
    c = orc.basis_state(2, [1, 0])
    assert orc.apply_gates(2, c, [(2, 0.0, [0, 1])])[3] == 1
    with pytest.raises(ValueError):
        orc.apply_gates(2, c, [(0, 0.0, [2])])
    with pytest.raises(ValueError):
        orc.apply_gates(2, c, [(2, 0.0, [0, 0])])


def test_adam_golden(orc):
    # test_vqe.cpp:119-138
    t, m, v, s = orc.adam_step([0.0], [0.0], 0, [1.0], [0.0])
    assert abs(t[0] - (-0.009999999900000002)) < 1e-15 and s == 1
    t0, *_ = orc.adam_step([0.0], [0.0], 0, [0.0], [0.3])
    assert t0[0] == 0.3


def test_counters_golden(orc):
    # test_vqe.cpp:171-180 and :228-236
    h = orc.build_h2_hamiltonian(0.7414)
    r = orc.run_vqe(h, tol=1e3)
    assert r["iterations_run"] == 0 and len(r["trajectory"]) == 1 and r["circuit_evaluations"] == 3
    r = orc.run_vqe(orc.build_h2_hamiltonian(0.9), max_iter=5)
    assert r["circuit_evaluations"] == 5 * 3 + 1


def test_chunks_golden(orc):
    # test_sweep.cpp:43-78 (sizes + exhaustive rule)
    sizes = lambda n, p: [e - b for b, e in orc.split_chunks(n, p)]  # noqa: E731
    assert sizes(100, 3) == [34, 33, 33]
    assert sizes(100, 32) == [4] * 4 + [3] * 28
    assert sizes(2, 4) == [1, 1, 0, 0]
    for n in range(0, 129, 7):
        for p in range(1, 65, 5):
            ch = orc.split_chunks(n, p)
            cur = 0
            for c, (b, e) in enumerate(ch):
                assert b == cur and e - b == ((n - c + p - 1) // p if c < n else 0)
                cur = e
            assert cur == n


def test_bond_grid_golden(orc):
    # test_sweep.cpp:25-41
    g = orc.bond_grid(0.5, 2.0, 7)
    assert g[0] == 0.5 and g[-1] == 2.0
    assert np.allclose(np.diff(g), 0.25, atol=1e-12)
    assert list(orc.bond_grid(0.7414, 0.7414, 1)) == [0.7414]
    with pytest.raises(ValueError):
        orc.bond_grid(1.0, 0.5, 4)
    with pytest.raises(ValueError):
        orc.bond_grid(0.5, 1.0, 0)


def test_nan_hamiltonian_message(orc):
    # test_vqe.cpp:238-254
    h = Ham(4, [(complex(float("nan"), 0.0), [])])
    with pytest.raises(RuntimeError, match="non-finite energy at iteration"):
        orc.run_vqe(h)


# ---------------------------------------------------------------- vs _ref
def test_oracle_matches_reference_hamiltonians_bitwise(orc, ref):
    for d in [0.05, 0.1, 0.4, 0.7414, 1.3, 2.2, 3.0, 7.5, 10.0]:
        a, b = orc.build_h2_hamiltonian(d), ref.build_h2_hamiltonian(d)
        assert a.terms == b.terms, d
    with pytest.raises(ArithmeticError, match="outside"):
        orc.build_h2_hamiltonian(0.01)
    with pytest.raises(ArithmeticError, match="outside"):
        ref.build_h2_hamiltonian(0.01)


def test_oracle_matches_reference_gates_expectation_bitwise(orc, ref):
    rng = np.random.default_rng(7)
    pr = random.Random(8)
    for n in [1, 2, 4, 7, 9]:
        psi = random_state(rng, n)
        gates = []
        for _ in range(30):
            k = pr.randint(0, 3 if n >= 4 else (2 if n >= 2 else 1))
            ws = pr.sample(range(n), [1, 1, 2, 4][k])
            gates.append((k, pr.uniform(-3.14, 3.14), ws))
        a, b = orc.apply_gates(n, psi, gates), ref.apply_gates(n, psi, gates)
        assert np.array_equal(a, b)
        h = ref.canonicalize(random_hamiltonian(pr, n, 16))
        assert orc.canonicalize(random_hamiltonian(random.Random(3), n, 16)).terms == \
            ref.canonicalize(random_hamiltonian(random.Random(3), n, 16)).terms
        assert orc.expectation(n, a, h) == ref.expectation(n, a, h)


def test_oracle_matches_reference_vqe_and_sweep_bitwise(orc, ref):
    for d in [0.7414, 2.6]:
        h = ref.build_h2_hamiltonian(d)
        a, b = orc.run_vqe(h), ref.run_vqe(h)
        assert np.array_equal(a["trajectory"], b["trajectory"]) and np.array_equal(a["theta"], b["theta"])
        a, b = orc.run_vqe(h, max_iter=5000, tol=1e-8), ref.run_vqe(h, max_iter=5000, tol=1e-8)
        assert a["iterations_run"] == b["iterations_run"]
    for n in [3, 5]:
        h = ref.build_tfim(n, 1.0, 1.0)
        assert orc.build_tfim(n, 1.0, 1.0).terms == h.terms
        assert orc.build_z_sum(n).terms == ref.build_z_sum(n).terms
        a = orc.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=4, init=[0.1] * (2 * n))
        b = ref.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=4, init=[0.1] * (2 * n))
        assert np.array_equal(a["trajectory"], b["trajectory"])
    s_o = orc.run_sweep(0.5, 2.0, 8, max_iter=25)
    s_r = ref.run_sweep(0.5, 2.0, 8, workers=3, max_iter=25)
    assert np.array_equal(s_o["energy"], s_r["energy"]) and np.array_equal(s_o["iterations"], s_r["iterations"])


# ------------------------------------------------------ vs committed fixtures
def test_oracle_matches_golden_fixtures(orc, golden):
    g = golden("h2_hamiltonians.json")
    for d, hj in g["hamiltonians"].items():
        want = Ham.from_text(4, hj["text"])
        got = orc.build_h2_hamiltonian(float(d))
        assert got.terms == want.terms, d
        assert orc.hartree_fock(float(d))["hf_energy"] == g["hartree_fock"][d]["hf_energy"]
    p = golden("pes_default.json")
    s = orc.run_sweep()
    assert list(s["bond"]) == p["bond"]
    assert list(s["energy"]) == p["energy"]
    assert list(s["iterations"]) == p["iterations"]
    t = p["tol_mode"]
    s = orc.run_sweep(max_iter=5000, tol=1e-8)
    assert list(s["iterations"]) == t["iterations"]
    c = golden("gates_expectation.json")["cases"][0]
    psi = np.array([complex(*x) for x in c["psi"]])
    out = orc.apply_gates(c["n"], psi, [tuple(x) for x in c["gates"]])
    assert np.array_equal(out, np.array([complex(*x) for x in c["out"]]))


def test_reference_pes_properties(golden):
    # acceptance criterion 2 (acceptance_main.cpp:112-132): argmin in
    # [0.70, 0.78] A, E within 0.005 of -1.137
    p = golden("pes_default.json")
    i = int(np.argmin(p["energy"]))
    assert 0.70 <= p["bond"][i] <= 0.78 and abs(p["energy"][i] + 1.137) < 0.005
    assert all(it == 200 for it in p["iterations"])


# ----------------------------------------- dense embedding (independent)
def _small_gate(kind, angle):
    """Local unitaries of tests/oracles/dense_gates.hpp:30-67 (wire k = local
    bit w-1-k) plus SingleExcitation, the engine's appended kind: the
    DoubleExcitation Givens restricted to |10>,|01> (local indices 2, 1)."""
    c, s = math.cos(0.5 * angle), math.sin(0.5 * angle)
    if kind == 0:
        return np.array([[0, 1], [1, 0]], dtype=complex)
    if kind == 1:
        return np.array([[c, -s], [s, c]], dtype=complex)
    if kind == 2:
        m = np.eye(4, dtype=complex)
        m[2, 2] = m[3, 3] = 0
        m[2, 3] = m[3, 2] = 1
        return m
    if kind == 3:
        m = np.eye(16, dtype=complex)
        m[12, 12], m[12, 3], m[3, 12], m[3, 3] = c, -s, s, c
        return m
    m = np.eye(4, dtype=complex)
    m[2, 2], m[2, 1], m[1, 2], m[1, 1] = c, -s, s, c
    return m


def _embed(kind, angle, wires, n):
    """dense_gates.hpp:70-101 embed_gate: the full 2^n unitary by index
    arithmetic (qubit 0 = most significant bit)."""
    small = _small_gate(kind, angle)
    w = len(wires)
    dim = 1 << n
    mask = 0
    for q in wires:
        mask |= 1 << (n - 1 - q)

    def loc(i):
        return sum(((i >> (n - 1 - q)) & 1) << (w - 1 - k) for k, q in enumerate(wires))

    full = np.zeros((dim, dim), dtype=complex)
    for i in range(dim):
        for j in range(dim):
            if (i & ~mask) == (j & ~mask):
                full[i, j] = small[loc(i), loc(j)]
    return full


@pytest.mark.parametrize("n", [2, 4, 6])
def test_single_excitation_oracle_vs_dense_embedding(orc, n):
    """The SingleExcitation restatement (vqf_oracle.c ORC_SE) against the
    dense embedding, in the style of test_statevector.cpp:150-166; DE and
    the reference kinds as a control of the embedding itself."""
    rng = np.random.default_rng(20260802 + n)
    pr = random.Random(n)
    for _ in range(20):
        kind = pr.choice([4, 4, 0, 1, 2] + ([3] if n >= 4 else []))
        wires = pr.sample(range(n), [1, 1, 2, 4, 2][kind])
        angle = pr.uniform(-3.2, 3.2)
        psi = random_state(rng, n)
        want = _embed(kind, angle, wires, n) @ psi
        got = orc.apply_gates(n, psi, [(kind, angle, wires)])
        assert np.max(np.abs(got - want)) < 1e-12
    # |10> -> cos|10> + sin|01>: the engine's convention (DE's, on two wires)
    e = orc.apply_gates(2, np.array([0, 0, 1, 0], dtype=complex), [(4, 0.6, [0, 1])])
    assert abs(e[2] - math.cos(0.3)) < 1e-15 and abs(e[1] - math.sin(0.3)) < 1e-15


def test_reference_fixtures_are_seeded(ref):
    """ref_random_hamiltonian / ref_random_state are test_helpers.hpp's own
    generators (mt19937): deterministic, normalised, the documented shape."""
    h = ref.random_hamiltonian(20260804, 6, 32)
    assert len(h.terms) == 32 and all(c.imag == 0 and -2 <= c.real <= 2 for c, _ in h.terms)
    assert ref.random_hamiltonian(20260804, 6, 32).terms == h.terms
    a = ref.random_state(20260802, 5)
    assert abs(np.vdot(a, a).real - 1) < 1e-14 and np.array_equal(a, ref.random_state(20260802, 5))
