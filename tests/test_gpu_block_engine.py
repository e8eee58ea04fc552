"""GPU parity of the shared-memory VQE engine (csrc/vqe_block.cu): one
cooperative launch per run_vqe for hardware-efficient registers of 4..14
qubits (complex128) / 4..15 (complex64).  Compared with the reference's own
run_vqe (oracle/_ref, vqe.hpp:194-254): trajectories, final energies and
parameters within 1e-10 Ha (fp64) / 1e-5 (fp32), identical iteration and
circuit-evaluation counts, the reference's error messages, and the HBM
engine on the same problems (VQF_ENGINE override)."""
from __future__ import annotations

import random

import numpy as np
import pytest

from oracle.oracle import Ham, random_hamiltonian

pytestmark = pytest.mark.gpu

E_TOL = 1e-10
F32_TOL = 1e-5


def to_v(V, h: Ham):
    return V.QubitHamiltonian(h.n_qubits, [V.PauliTerm(c, a) for c, a in h.terms])


def hams(ref, n):
    tf = ref.build_tfim(n, 1.0, 0.7)
    rh = random_hamiltonian(random.Random(20260804 + n), n, 16)
    return {"tfim": tf, "random16": ref.canonicalize(rh)}


@pytest.mark.parametrize("n", [4, 6, 8, 10, 12, 13, 14])
def test_block_engine_run_vqe_matches_reference(gpu, ref, n, monkeypatch):
    """4..13 qubits: state in shared memory; 14: in an L2-resident global
    buffer per CTA."""
    V = gpu
    monkeypatch.setenv("VQF_ENGINE", "block")  # n = 4, 5 default to the warp engine
    hea = V.AnsatzSpec.hardware_efficient(2)
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=5)
    init = [0.1] * (2 * n)
    for name, h in hams(ref, n).items():
        want = ref.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=5, init=init)
        for method in ("shift", "adjoint"):
            r = V.run_vqe(to_v(V, h), hea, cfg, init, method=method)
            assert r.iterations_run == want["iterations_run"] == 5, name
            assert r.circuit_evaluations == want["circuit_evaluations"], name
            assert len(r.trajectory) == len(want["trajectory"])
            assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL, name
            assert abs(r.energy - want["energy"]) < E_TOL and r.energy == r.trajectory[-1]
            assert np.max(np.abs(np.array(r.theta) - want["theta"])) < 1e-9, name


@pytest.mark.parametrize("n,layers,iters", [(6, 8, 3), (9, 7, 2), (11, 1, 4)])
def test_block_engine_many_circuits_and_layers(gpu, ref, n, layers, iters):
    """2P + 1 above the co-resident grid (CTAs loop over circuits) and
    single-layer frames."""
    V = gpu
    h = ref.build_tfim(n, 0.8, 1.1)
    # generic angles: a parameter whose gradient vanishes by symmetry turns
    # rounding-level differences into O(lr) Adam steps (ill-conditioned)
    init = list(np.random.default_rng(n * layers).uniform(-1.0, 1.0, layers * n))
    want = ref.run_vqe(h, kind=1, layers=layers, lr=0.03, max_iter=iters, init=init)
    r = V.run_vqe(to_v(V, h), V.AnsatzSpec.hardware_efficient(layers), V.AdamConfig(learning_rate=0.03, max_iterations=iters),
                  init)
    assert r.circuit_evaluations == want["circuit_evaluations"]
    assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL


def test_block_engine_tolerance_mode_and_zero_iterations(gpu, ref):
    V = gpu
    n = 6
    h = ref.build_tfim(n, 1.0, 0.7)
    hea = V.AnsatzSpec.hardware_efficient(1)
    init = [0.3] * n
    want = ref.run_vqe(h, kind=1, layers=1, lr=0.05, max_iter=400, tol=2e-3, init=init)
    assert 0 < want["iterations_run"] < 400
    r = V.run_vqe(to_v(V, h), hea, V.AdamConfig(learning_rate=0.05, max_iterations=400, gradient_tolerance=2e-3), init)
    assert r.iterations_run == want["iterations_run"]
    assert r.circuit_evaluations == want["circuit_evaluations"]
    assert len(r.trajectory) == r.iterations_run + 1
    assert abs(r.energy - want["energy"]) < E_TOL
    r0 = V.run_vqe(to_v(V, h), hea, V.AdamConfig(max_iterations=0), init)
    w0 = ref.run_vqe(h, kind=1, layers=1, max_iter=0, init=init)
    assert r0.iterations_run == 0 and r0.circuit_evaluations == 1 and r0.theta == init
    assert abs(r0.energy - w0["energy"]) < E_TOL


def test_block_engine_errors(gpu, ref):
    V = gpu
    n = 7
    hea = V.AnsatzSpec.hardware_efficient(2)
    bad = V.QubitHamiltonian(n, [V.PauliTerm(complex(float("nan"), 0.0), [(0, 3)])])
    with pytest.raises(RuntimeError, match=r"non-finite energy at iteration 0; theta = 0\.000000"):
        V.run_vqe(bad, hea)
    nh = V.QubitHamiltonian(n, [V.PauliTerm(1.0, [(0, 1)]), V.PauliTerm(0.5j, [(3, 3)])])
    with pytest.raises(RuntimeError, match="imaginary residue"):
        V.run_vqe(nh, hea, V.AdamConfig(max_iterations=3), [0.2] * (2 * n))
    h = to_v(V, ref.build_tfim(n, 1.0, 1.0))
    with pytest.raises(ValueError, match="initial parameter count mismatch"):
        V.run_vqe(h, hea, V.AdamConfig(), [0.1])
    # back-to-back runs are bitwise repeatable (fixed-order reductions)
    a = V.run_vqe(h, hea, V.AdamConfig(max_iterations=20), [0.1] * (2 * n))
    b = V.run_vqe(h, hea, V.AdamConfig(max_iterations=20), [0.1] * (2 * n))
    assert a.trajectory == b.trajectory and a.theta == b.theta


@pytest.mark.parametrize("n", [8, 11])
def test_block_engine_equals_hbm_engine(gpu, ref, n, monkeypatch):
    V = gpu
    h = to_v(V, hams(ref, n)["random16"])
    hea = V.AnsatzSpec.hardware_efficient(2)
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=6)
    init = [0.2] * (2 * n)
    monkeypatch.setenv("VQF_ENGINE", "block")
    rb = V.run_vqe(h, hea, cfg, init)
    monkeypatch.setenv("VQF_ENGINE", "hbm")
    rh = V.run_vqe(h, hea, cfg, init)
    assert np.max(np.abs(np.array(rb.trajectory) - rh.trajectory)) < 1e-12
    assert np.max(np.abs(np.array(rb.theta) - rh.theta)) < 1e-11


@pytest.mark.parametrize("n", [6, 10, 14, 15])
def test_block_engine_fp32(gpu, ref, n):
    V = gpu
    h = ref.build_tfim(n, 1.0, 0.7)
    init = [0.1] * (2 * n)
    want = ref.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=5, init=init)
    r = V.run_vqe(to_v(V, h), V.AnsatzSpec.hardware_efficient(2), V.AdamConfig(learning_rate=0.05, max_iterations=5), init,
                  dtype="f32")
    # complex64 storage rounds every amplitude once per pass; relative bar
    # once |E| > 1, as test_f32_run_vqe_fixed_iterations (test_gpu_parity.py)
    bar = F32_TOL * np.maximum(1.0, np.abs(want["trajectory"]))
    assert np.all(np.abs(np.array(r.trajectory) - want["trajectory"]) < bar)
    assert r.circuit_evaluations == want["circuit_evaluations"]


def test_scaling_study_mid_widths_match_reference(gpu, ref):
    """run_scaling_study (sweep.hpp:265-307) at the config-3 widths the
    engine holds (4..14)."""
    V = gpu
    widths = [4, 6, 8, 10, 12, 13, 14]
    recs = V.run_scaling_study(V.ScalingConfig(qubits=widths))
    want = ref.run_scaling_study(widths)
    for r, w in zip(recs, want):
        assert r["n_qubits"] == w["n_qubits"] and r["iterations_run"] == w["iterations_run"]
        assert abs(r["final_energy"] - w["final_energy"]) < E_TOL


def test_run_vqe_batch_hea_routes_per_problem(gpu, ref):
    """run_vqe_batch with a 5-qubit HEA(2) (32 amplitudes per lane would
    spill the one-warp engine): each problem runs on the shared-memory
    engine and matches run_vqe and the reference."""
    V = gpu
    n = 5
    hs = [ref.build_tfim(n, 1.0, f) for f in (0.5, 0.9, 1.3)]
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=6)
    rs = V.run_vqe_batch([to_v(V, h) for h in hs], V.AnsatzSpec.hardware_efficient(2), cfg)
    for h, r in zip(hs, rs):
        want = ref.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=6)
        assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL
        assert r.circuit_evaluations == want["circuit_evaluations"]
