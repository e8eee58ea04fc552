"""CPU: the C-ABI library loads, exports every symbol include/vqf_b200.h
declares, and its host-only functions (no GPU involved) match the oracle:
bond_grid / split_chunks / effective_workers (sweep.hpp:68-119), adam_step
(vqe.hpp:152-174), canonicalize (pauli.hpp:180-201), TFIM / Z-sum builders
(sweep.hpp:209-235) and the H2 Hamiltonian (chem.hpp:473)."""
from __future__ import annotations

import ctypes
import os
import random
import re

import numpy as np
import pytest

from oracle.oracle import Ham, random_hamiltonian

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vqf_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vqf_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(V):
    names = declared_functions()
    assert len(names) >= 30
    lib = ctypes.CDLL(V.lib._name)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2601_09951_b200 import _capi

    bound = {s[0] for s in _capi.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound


def test_library_is_sm100a_only(V):
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", V.lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_version_and_memory_estimate(V):
    assert b"sm_100a" in V.lib.vqf_version()
    # test_statevector.cpp:92-94
    assert V.memory_estimate(4) == 256
    assert V.memory_estimate(20) == 16 * 1024 * 1024
    assert V.memory_estimate(26) == 1024 ** 3


def test_n_parameters(V):
    assert V.n_parameters(V.AnsatzSpec.h2_double_excitation(), 4) == 1
    assert V.n_parameters(V.AnsatzSpec.hardware_efficient(3), 5) == 15


def test_bond_grid_bitwise(V, orc):
    for args in [(0.1, 3.0, 100), (0.5, 2.0, 7), (0.7414, 0.7414, 1), (0.7414, 0.7414, 3), (0.1, 3.0, 2)]:
        assert V.bond_grid(*args) == list(orc.bond_grid(*args))
    with pytest.raises(ValueError, match="d_max < d_min"):
        V.bond_grid(1.0, 0.5, 4)
    with pytest.raises(ValueError, match="grid needs"):
        V.bond_grid(0.5, 1.0, 0)


def test_split_chunks_exhaustive(V):
    # test_sweep.cpp:59-76
    for n in range(0, 129):
        for p in range(1, 65):
            ch = V.split_chunks(n, p)
            assert len(ch) == p
            cur = 0
            for c, (b, e) in enumerate(ch):
                assert b == cur and e - b == ((n - c + p - 1) // p if c < n else 0)
                cur = e
            assert cur == n
    with pytest.raises(ValueError):
        V.split_chunks(10, 0)


def test_effective_workers(V, monkeypatch):
    # test_sweep.cpp:80-99
    monkeypatch.delenv("VQE_FORGE_THREADS", raising=False)
    assert V.effective_workers(8) == 8
    monkeypatch.setenv("VQE_FORGE_THREADS", "2")
    assert V.effective_workers(8) == 2 and V.effective_workers(1) == 1
    for bad in ["abc", "0", "-3", "2x"]:
        monkeypatch.setenv("VQE_FORGE_THREADS", bad)
        assert V.effective_workers(8) == 8
    monkeypatch.delenv("VQE_FORGE_THREADS")
    with pytest.raises(ValueError):
        V.effective_workers(0)


def test_adam_step_bitwise(V, orc):
    cfg = V.AdamConfig()
    t, s = V.adam_step(V.AdamState.zeros(1), [1.0], [0.0], cfg)
    assert t[0] == -0.009999999900000002 and s.step == 1  # test_vqe.cpp:129
    rng = np.random.default_rng(5)
    m, v, g, th = (rng.standard_normal(7) for _ in range(4))
    v = np.abs(v)
    for step in [0, 1, 17, 199]:
        a = V.adam_step(V.AdamState(list(m), list(v), step), list(g), list(th), cfg)
        b = orc.adam_step(m, v, step, g, th)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1].m, b[1]) and np.array_equal(a[1].v, b[2])
    with pytest.raises(ValueError):
        V.adam_step(V.AdamState.zeros(1), [1.0, 2.0], [0.0], cfg)


def _to_orc(h):
    return Ham(h.n_qubits, [(t.coefficient, t.axes) for t in h.terms])


def test_canonicalize_matches_oracle(V, orc):
    for seed in range(6):
        pr = random.Random(seed)
        n = pr.randint(1, 9)
        raw = random_hamiltonian(pr, n, pr.randint(1, 40), real=seed % 2 == 0)
        # duplicate some terms so merging is exercised
        raw.terms += raw.terms[: len(raw.terms) // 2]
        mine = V.canonicalize(V.QubitHamiltonian(n, [V.PauliTerm(c, a) for c, a in raw.terms]))
        assert _to_orc(mine).terms == orc.canonicalize(raw).terms
    with pytest.raises(ValueError, match="explicit identity"):
        V.canonicalize(V.QubitHamiltonian(2, [V.PauliTerm(1.0, [(0, 0)])]))
    with pytest.raises(ValueError, match="duplicate qubit"):
        V.canonicalize(V.QubitHamiltonian(2, [V.PauliTerm(1.0, [(0, 1), (0, 3)])]))


def test_builders_match_oracle(V, orc):
    for n in [2, 4, 5, 9, 20]:
        assert _to_orc(V.build_tfim(n, 1.0, 1.0)).terms == orc.build_tfim(n, 1.0, 1.0).terms
        assert _to_orc(V.build_z_sum(n)).terms == orc.build_z_sum(n).terms
    assert len(V.build_tfim(5, 1.0, 1.0).terms) == 9  # test_sweep.cpp:177-178
    assert len(V.build_tfim(4, 1.0, 0.0).terms) == 3


def test_h2_hamiltonian_matches_golden(V, golden):
    """Host build of chem.hpp:473 against the reference's fixtures: same
    strings in canonical order, coefficients within 1e-13."""
    g = golden("h2_hamiltonians.json")
    for d, hj in g["hamiltonians"].items():
        want = Ham.from_text(4, hj["text"])
        got = _to_orc(V.build_h2_hamiltonian(float(d)))
        assert [t[1] for t in got.terms] == [t[1] for t in want.terms], d
        for (cg, _), (cw, _) in zip(got.terms, want.terms):
            assert abs(cg - cw) <= 1e-13, (d, cg, cw)  # test_chem.cpp:244 uses 1e-12
        hf = V.run_hartree_fock(float(d))
        assert abs(hf["hf_energy"] - g["hartree_fock"][d]["hf_energy"]) < 1e-13


def test_h2_errors(V):
    with pytest.raises(V.BondLengthOutOfRange, match=r"bond length 0\.010000 angstrom outside \[0\.050000, 10\.000000\]"):
        V.build_h2_hamiltonian(0.01)
    with pytest.raises(V.BondLengthOutOfRange):
        V.build_h2_hamiltonian(10.5)
    assert len(V.build_h2_hamiltonian(0.05).terms) == 15
    assert len(V.build_h2_hamiltonian(10.0).terms) >= 1


def test_speedup_arithmetic(V):
    # test_sweep.cpp:145-175
    assert abs(V.measured_speedup(143.80, 5.04) - 28.53) < 0.01
    assert abs(V.amdahl_speedup(0.05, 4) - 3.4783) < 1e-4
    with pytest.raises(ValueError):
        V.measured_speedup(0.0, 1.0)
    with pytest.raises(ValueError):
        V.amdahl_speedup(1.1, 4)


def test_expectation_plan_packs_flip_groups(V):
    """Host plan of the expectation (no GPU): TFIM's n single-X flip groups
    share register passes four high bits at a time plus every lane-bit
    group; a Z-only sum is one diagonal pass; dense random strings fall back
    to one pass per group."""
    for n in [9, 10]:  # below the 2^11-amplitude gathered tile: register passes
        p = V.expectation_plan(V.build_tfim(n, 1.0, 1.0))
        assert p["flip_groups"] == n
        high = n - 5  # X on index bits 5..n-1
        assert p["multi_passes"] == -(-high // 4)
        assert p["state_passes"] == 1 + p["multi_passes"]
    # from 11 qubits: gathered-tile passes (expect_tile.cu), up to 3 phases x 4
    # single-bit groups each, windows of contiguous high bits; the fp64 plan
    # folds the n - 1 real Z Z terms into one of them (no diagonal pass)
    for n, passes in [(11, 1), (12, 2), (20, 3), (26, 3), (30, 4), (33, 4)]:
        p = V.expectation_plan(V.build_tfim(n, 1.0, 1.0))
        assert p["flip_groups"] == n
        assert p["multi_passes"] == passes, (n, p)
        assert p["state_passes"] == passes
    assert V.expectation_plan(V.build_z_sum(24)) == {"state_passes": 1, "flip_groups": 0, "multi_passes": 0}
    # below 9 qubits there are no register passes: one pass per group
    p = V.expectation_plan(V.build_tfim(6, 1.0, 1.0))
    assert p == {"state_passes": 7, "flip_groups": 6, "multi_passes": 0}
    rh = random_hamiltonian(random.Random(20260804), 26, 32)
    h = V.canonicalize(V.QubitHamiltonian(26, [V.PauliTerm(c, a) for c, a in rh.terms]))
    p = V.expectation_plan(h)
    assert p["flip_groups"] >= 28 and p["multi_passes"] <= 2
    assert p["flip_groups"] - 2 <= p["state_passes"] <= p["flip_groups"] + 1


def test_circuit_plan_fuses_hea_layers(V):
    """Host plan of apply_circuit (no GPU): one HEA layer (RY on every wire +
    CNOT chain, vqe.hpp:81-93) needs far fewer HBM passes than gates; the
    scheduler advances the CNOT chain five wires per pass (six gathered high
    bits) and composes the gates into few register ops per pass."""
    for n in [12, 20, 26, 30, 33]:
        layer = [V.Gate.ry(0.1, q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
        p = V.circuit_plan(n, layer)
        assert p["passes"] <= 1 + max(0, -(-(n - 6 - 1) // 5)), (n, p)
        assert p["fused_ops"] <= len(layer) // 2
    assert V.circuit_plan(10, [V.Gate.ry(0.3, 0)]) == {"passes": 1, "fused_ops": 0}
    with pytest.raises(ValueError, match="exceeds register"):
        V.circuit_plan(4, [V.Gate.ry(0.1, 5), V.Gate.ry(0.1, 0)])
