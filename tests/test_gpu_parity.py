"""GPU parity: the sm_100a engine (through the C ABI) against the CPU oracle
and the reference's golden fixtures.  Bar (BASELINE.json north_star):
energies within 1e-10 Ha in fp64 (1e-5 in fp32), bit-identical iteration
counts and bond grid, results independent of GPU/worker count.
Amplitudes: 1e-12 per amplitude (the reference's own test tolerance,
test_statevector.cpp:150-166)."""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

from oracle.oracle import Ham, random_hamiltonian, random_state
from vqf_helpers import ham_from_text

pytestmark = pytest.mark.gpu

E_TOL = 1e-10   # fp64 energies (north_star)
A_TOL = 1e-12   # amplitudes (test_statevector.cpp:166)
TH_TOL = 1e-12  # optimised parameters (measured: <= 8e-15 on the default PES)


def to_v(V, h: Ham):
    return V.QubitHamiltonian(h.n_qubits, [V.PauliTerm(c, a) for c, a in h.terms])


def rand_gates(pr, n, count, kinds=(0, 1, 2, 3, 4)):
    out = []
    for _ in range(count):
        k = pr.choice([k for k in kinds if [1, 1, 2, 4, 2][k] <= n])
        ws = pr.sample(range(n), [1, 1, 2, 4, 2][k])
        out.append((k, pr.uniform(-3.14, 3.14), ws))
    return out


def gpu_gate(V, k, angle, ws):
    return V.Gate(k, angle, tuple(ws))


# ------------------------------------------------------------ state vector
def test_basis_state_and_reset(gpu):
    V = gpu
    psi = V.basis_state(4, [1, 1, 0, 0])
    a = psi.amplitudes
    assert a[12] == 1 and np.count_nonzero(a) == 1
    assert V.basis_state(2, [0, 1]).amplitudes[1] == 1
    with pytest.raises(ValueError, match="bit count"):
        V.basis_state(2, [0, 1, 0])
    z = V.StateVector(3)
    assert z.amplitudes[0] == 1 and abs(z.norm() - 1.0) < 1e-15


@pytest.mark.parametrize("n", [4, 5, 7, 10, 13])
def test_gates_match_oracle(gpu, orc, n):
    V = gpu
    rng = np.random.default_rng(100 + n)
    pr = random.Random(200 + n)
    psi0 = random_state(rng, n)
    gates = rand_gates(pr, n, 40, kinds=(0, 1, 2, 3, 4))  # SingleExcitation: vqf_oracle.c ORC_SE
    want = orc.apply_gates(n, psi0, gates)
    psi = V.StateVector(n)
    psi.amplitudes = psi0
    V.apply_circuit(psi, [gpu_gate(V, *g) for g in gates])
    got = psi.amplitudes
    assert np.max(np.abs(got - want)) < A_TOL
    # per-gate too (each kind on every wire position class)
    psi.amplitudes = psi0
    cur = psi0
    for g in gates[:8]:
        V.apply_gate(psi, gpu_gate(V, *g))
        cur = orc.apply_gates(n, cur, [g])
        assert np.max(np.abs(psi.amplitudes - cur)) < A_TOL


@pytest.mark.parametrize("n,dtype", [(3, "f64"), (4, "f32"), (5, "f64"), (12, "f64"), (13, "f32"), (16, "f64"),
                                     (17, "f32"), (19, "f64")])
def test_fused_circuit_equals_per_gate(gpu, n, dtype):
    # apply_circuit (k_tile: TMA-swizzled tiles, gates fused into register
    # ops of <= 4 local bits) against one apply_gate launch per gate, on
    # every gate kind with random wires (low and high index bits)
    V = gpu
    pr = random.Random(9000 + n)
    gates = [gpu_gate(V, *g) for g in rand_gates(pr, n, 120)]
    psi0 = random_state(np.random.default_rng(n), n)
    a, b = V.StateVector(n, dtype=dtype), V.StateVector(n, dtype=dtype)
    a.amplitudes = psi0
    b.amplitudes = psi0
    V.apply_circuit(a, gates)
    for g in gates:
        V.apply_gate(b, g)
    tol = 1e-12 if dtype == "f64" else 2e-5
    assert np.max(np.abs(a.amplitudes - b.amplitudes)) < tol


@pytest.mark.parametrize("n,batch", [(22, 1), (14, 3)])
def test_fused_wide_circuits_and_batches(gpu, n, batch):
    # larger registers: many passes, 4-bit DoubleExcitation ops (wide kernel),
    # 3-bit tensor-core ops and permutation passes in one circuit; batched
    # states (one CTA row per entry) against the per-gate kernels
    V = gpu
    pr = random.Random(777 + n)
    gates = [gpu_gate(V, *g) for g in rand_gates(pr, n, 150)]
    gates += [V.Gate.cnot(q, q + 1) for q in range(n - 1)] + [V.Gate.double_excitation(0.3, n - 4, n - 1, 0, 2)]
    rng = np.random.default_rng(n)
    psi0 = np.concatenate([random_state(rng, n) for _ in range(batch)])
    a, b = V.StateVector(n, batch=batch), V.StateVector(n, batch=batch)
    a.amplitudes = psi0
    b.amplitudes = psi0
    V.apply_circuit(a, gates)
    for g in gates:
        V.apply_gate(b, g)
    assert np.max(np.abs(a.amplitudes - b.amplitudes)) < 1e-12


@pytest.mark.parametrize("n,dtype,batch", [(20, "f64", 1), (21, "f32", 1), (16, "f64", 3), (17, "f32", 2)])
def test_fused_window_boxes_equal_run_boxes(gpu, n, dtype, batch, monkeypatch):
    # passes whose gathered bits form one window move each tile as one 5-d
    # TMA box (tile map); VQF_TILE_NO_WINDOW forces one box per run.  Same
    # arithmetic, different data movement: bitwise equal, batched entries too
    V = gpu
    pr = random.Random(5150 + n)
    hea = [V.Gate.ry(0.1 * (q + 1), q) for q in range(n)] + [V.Gate.cnot(q, q + 1) for q in range(n - 1)]
    gates = hea + [gpu_gate(V, *g) for g in rand_gates(pr, n, 60)] + hea
    rng = np.random.default_rng(n + 11)
    psi0 = np.concatenate([random_state(rng, n) for _ in range(batch)])
    out = []
    for no_window in (False, True):
        if no_window:
            monkeypatch.setenv("VQF_TILE_NO_WINDOW", "1")
        s = V.StateVector(n, dtype=dtype, batch=batch)
        s.amplitudes = psi0
        V.apply_circuit(s, gates)
        out.append(s.amplitudes)
    assert np.array_equal(out[0], out[1])
    ref = V.StateVector(n, dtype=dtype, batch=batch)
    ref.amplitudes = psi0
    for g in gates:
        V.apply_gate(ref, g)
    assert np.max(np.abs(out[0] - ref.amplitudes)) < (1e-12 if dtype == "f64" else 2e-5)


@pytest.mark.parametrize("n,dtype", [(5, "f64"), (12, "f64"), (16, "f64"), (19, "f32")])
def test_fused_permutation_passes(gpu, n, dtype):
    # X / CNOT-only circuits: every tile pass is an affine index map applied
    # in the write-back (no register ops); against one launch per gate
    V = gpu
    pr = random.Random(4000 + n)
    gates = [gpu_gate(V, *g) for g in rand_gates(pr, n, 80, kinds=(0, 2))]
    psi0 = random_state(np.random.default_rng(n + 7), n)
    a, b = V.StateVector(n, dtype=dtype), V.StateVector(n, dtype=dtype)
    a.amplitudes = psi0
    b.amplitudes = psi0
    V.apply_circuit(a, gates)
    for g in gates:
        V.apply_gate(b, g)
    assert np.array_equal(a.amplitudes, b.amplitudes)  # pure data movement: bitwise
    assert V.circuit_plan(n, gates, dtype)["fused_ops"] == 0


def test_gate_goldens(gpu, golden):
    V = gpu
    for c in golden("gates_expectation.json")["cases"]:
        n = c["n"]
        psi = V.StateVector(n)
        psi.amplitudes = np.array([complex(*x) for x in c["psi"]])
        V.apply_circuit(psi, [V.Gate(k, a, tuple(w)) for k, a, w in c["gates"]])
        want = np.array([complex(*x) for x in c["out"]])
        assert np.max(np.abs(psi.amplitudes - want)) < A_TOL
        h, _ = ham_from_text(V, n, c["hamiltonian"]["text"])
        assert abs(V.expectation(psi, h) - c["expectation_out"]) < E_TOL


def test_single_excitation_properties(gpu):
    """SingleExcitation (appended kind): Givens on |10>,|01>, angles add,
    norm preserved."""
    V = gpu
    psi = V.basis_state(2, [1, 0])
    V.apply_gate(psi, V.Gate.single_excitation(0.6, 0, 1))
    a = psi.amplitudes
    assert abs(a[2].real - math.cos(0.3)) < 1e-15 and abs(a[1].real - math.sin(0.3)) < 1e-15
    rng = np.random.default_rng(3)
    x = random_state(rng, 6)
    p, q = V.StateVector(6), V.StateVector(6)
    p.amplitudes = x
    q.amplitudes = x
    V.apply_circuit(p, [V.Gate.single_excitation(0.4, 1, 4), V.Gate.single_excitation(-1.1, 1, 4)])
    V.apply_gate(q, V.Gate.single_excitation(-0.7, 1, 4))
    assert np.max(np.abs(p.amplitudes - q.amplitudes)) < 1e-12
    assert abs(p.norm() - 1.0) < 1e-12


def test_gate_validation(gpu):
    V = gpu
    psi = V.StateVector(2)
    with pytest.raises(ValueError, match="exceeds register"):
        V.apply_gate(psi, V.Gate.pauli_x(2))
    with pytest.raises(ValueError, match="duplicate gate wire"):
        V.apply_gate(psi, V.Gate.cnot(0, 0))
    with pytest.raises(ValueError, match="exceeds register"):
        V.apply_gate(psi, V.Gate.double_excitation(1.0, 0, 1, 2, 3))
    with pytest.raises(ValueError, match="wire count"):
        V.apply_gate(psi, V.Gate(1, 0.1, (0, 1)))


@pytest.mark.parametrize("n", [1, 4, 6, 9, 11, 12, 14, 17])
def test_expectation_matches_oracle(gpu, orc, n):
    V = gpu
    rng = np.random.default_rng(300 + n)
    for trial in range(5):
        pr = random.Random(1000 * n + trial)
        h = orc.canonicalize(random_hamiltonian(pr, n, 12 if trial else 40, real=True))
        psi0 = random_state(rng, n)
        psi = V.StateVector(n)
        psi.amplitudes = psi0
        assert abs(V.expectation(psi, to_v(V, h)) - orc.expectation(n, psi0, h)) < E_TOL


def test_expectation_tfim_and_diagonal(gpu, orc):
    V = gpu
    for n in [2, 5, 11, 16]:
        h = orc.build_tfim(n, 1.0, 0.7)
        psi0 = random_state(np.random.default_rng(n), n)
        psi = V.StateVector(n)
        psi.amplitudes = psi0
        assert abs(V.expectation(psi, to_v(V, h)) - orc.expectation(n, psi0, h)) < E_TOL
    # test_statevector.cpp:185-196
    z = V.QubitHamiltonian(1, [V.PauliTerm(1.0, [(0, 3)])])
    assert abs(V.expectation(V.StateVector(1), z) - 1.0) < 1e-15
    ones = V.basis_state(4, [1, 1, 1, 1])
    assert abs(V.expectation(ones, V.build_z_sum(4)) + 4.0) < 1e-15
    with pytest.raises(ValueError, match="qubit count mismatch"):
        V.expectation(V.StateVector(2), V.QubitHamiltonian(3, [V.PauliTerm(1.0, [(0, 3)])]))


@pytest.mark.parametrize("n,n_terms", [(11, 30), (13, 60), (15, 150)])
def test_expectation_diagonal_factorised_pass(gpu, orc, n, n_terms):
    # Z-only strings exercise every split of the factorised diagonal pass:
    # support below bit 11, at/above bit 11, and straddling it with every
    # bits-8..10 pattern; 150 terms overflow the 64-term tables (fallback).
    V = gpu
    pr = random.Random(77 * n + n_terms)
    terms = []
    for t in range(n_terms):
        k = 1 + pr.randrange(min(n, 6))
        wires = sorted(pr.sample(range(n), k))
        terms.append((pr.uniform(-2, 2), [(w, 3) for w in wires]))
    terms += [(0.5, [(n - 1 - b, 3) for b in range(8, min(n, 11))]), (-0.25, [(0, 3), (n - 1, 3)])]
    h = orc.canonicalize(Ham(n, terms))
    psi0 = random_state(np.random.default_rng(n), n)
    psi = V.StateVector(n)
    psi.amplitudes = psi0
    assert abs(V.expectation(psi, to_v(V, h)) - orc.expectation(n, psi0, h)) < E_TOL


@pytest.mark.parametrize("n,n_terms", [(9, 40), (12, 120), (16, 300)])
def test_expectation_multi_group_passes(gpu, orc, n, n_terms):
    # few-body Pauli strings: most flip groups have <= 4 flip bits above the
    # lane bits and are packed into register-resident multi-group passes;
    # shared flips with different Z/Y patterns give multi-term groups, and
    # 300 terms open several passes (first fit) next to per-group fallbacks
    V = gpu
    pr = random.Random(4242 + n)
    terms = []
    for t in range(n_terms):
        k = 1 + pr.randrange(4)
        wires = sorted(pr.sample(range(n), k))
        terms.append((pr.uniform(-2, 2), [(w, 1 + pr.randrange(3)) for w in wires]))
    for t in range(n_terms // 10):  # repeat flips with other Z patterns
        c, axes = terms[pr.randrange(len(terms))]
        extra = [w for w in range(n) if w not in [q for q, _ in axes]]
        axes = sorted(axes + [(pr.choice(extra), 3)]) if extra else axes
        terms.append((pr.uniform(-1, 1), axes))
    h = orc.canonicalize(Ham(n, terms))
    psi0 = random_state(np.random.default_rng(n + 1), n)
    psi = V.StateVector(n)
    psi.amplitudes = psi0
    assert abs(V.expectation(psi, to_v(V, h)) - orc.expectation(n, psi0, h)) < E_TOL
    psi32 = V.StateVector(n, dtype="f32")
    psi32.amplitudes = psi0
    assert abs(V.expectation(psi32, to_v(V, h)) - orc.expectation(n, psi0, h)) < 1e-5 * max(1.0, len(terms) / 10)


def test_expectation_imaginary_residue_raises(gpu):
    V = gpu
    psi = V.StateVector(2)
    V.apply_gate(psi, V.Gate.ry(0.7, 0))
    h = V.QubitHamiltonian(2, [V.PauliTerm(1j, [])])  # non-Hermitian: <psi|iI|psi> = i
    with pytest.raises(RuntimeError, match="imaginary residue"):
        V.expectation(psi, h)


def test_norm_preserved_random_circuit(gpu):
    # test_statevector.cpp:168-175 at larger widths
    V = gpu
    pr = random.Random(20260803)
    for n in [4, 16, 22]:
        psi = V.StateVector(n)
        V.apply_circuit(psi, [gpu_gate(V, *g) for g in rand_gates(pr, n, 60)])
        assert abs(psi.norm() - 1.0) < 1e-10


def test_f32_state_within_tolerance(gpu, orc):
    V = gpu
    n = 12
    rng = np.random.default_rng(11)
    pr = random.Random(12)
    psi0 = random_state(rng, n)
    gates = rand_gates(pr, n, 30, kinds=(0, 1, 2, 3))
    h = orc.build_tfim(n, 1.0, 1.0)
    want = orc.expectation(n, orc.apply_gates(n, psi0, gates), h)
    psi = V.StateVector(n, dtype="f32")
    psi.amplitudes = psi0
    V.apply_circuit(psi, [gpu_gate(V, *g) for g in gates])
    assert abs(V.expectation(psi, to_v(V, h)) - want) < 1e-5


# -------------------------------------------------------------------- vqe
def test_prepare_ansatz_and_energy(gpu, orc, ref):
    V = gpu
    H2 = V.AnsatzSpec.h2_double_excitation()
    a = V.prepare_ansatz(H2, [math.pi], 4).amplitudes
    assert abs(a[3].real - 1) < 1e-15 and abs(a[12]) < 1e-15  # test_vqe.cpp:49-52
    for th in [-2.0, 0.3, 1.7]:
        a = V.prepare_ansatz(H2, [th], 4).amplitudes
        assert np.count_nonzero(np.delete(a, [3, 12])) == 0
    with pytest.raises(ValueError, match="parameter count"):
        V.prepare_ansatz(H2, [0.0, 0.0], 4)
    with pytest.raises(ValueError, match="requires 4 qubits"):
        V.prepare_ansatz(H2, [0.0], 6)
    hea = V.AnsatzSpec.hardware_efficient(2)
    th = np.random.default_rng(1).uniform(-3, 3, 12)
    assert np.max(np.abs(V.prepare_ansatz(hea, th, 6).amplitudes - orc.prepare_ansatz(1, 2, th, 6))) < A_TOL
    # test_vqe.cpp:82-89 E(0) = HF energy
    for d in [0.5, 0.7414, 1.6]:
        h = to_v(V, ref.build_h2_hamiltonian(d))
        assert abs(V.energy([0.0], h, H2) - ref.hartree_fock(d)["hf_energy"]) < E_TOL
    h = ref.build_tfim(6, 1.0, 1.0)
    assert abs(V.energy(th, to_v(V, h), hea) - orc.energy(1, 2, th, h)) < E_TOL


def test_gradient_matches_oracle(gpu, orc):
    V = gpu
    rng = np.random.default_rng(20260811)
    for d in [0.6, 1.3, 2.4]:
        h = orc.build_h2_hamiltonian(d)
        th = [rng.uniform(-3, 3)]
        g = V.gradient(th, to_v(V, h), V.AnsatzSpec.h2_double_excitation())
        assert abs(g[0] - orc.gradient(0, 0, th, h)[0]) < E_TOL
    h = orc.build_tfim(7, 1.0, 1.0)
    th = rng.uniform(-1, 1, 14)
    g = V.gradient(th, to_v(V, h), V.AnsatzSpec.hardware_efficient(2))
    assert np.max(np.abs(g - orc.gradient(1, 2, th, h))) < E_TOL
    # test_vqe.cpp:108-117
    g = V.gradient([0.0] * 4, V.build_z_sum(4), V.AnsatzSpec.hardware_efficient(1))
    assert np.max(np.abs(g)) < 1e-12


def test_run_vqe_h2_matches_golden(gpu, golden, ref):
    V = gpu
    g = golden("vqe_runs.json")["h2"]
    H2 = V.AnsatzSpec.h2_double_excitation()
    for d, want in g.items():
        h = to_v(V, ref.build_h2_hamiltonian(float(d)))
        r = V.run_vqe(h, H2)
        assert r.iterations_run == 200 and len(r.trajectory) == 201
        assert r.circuit_evaluations == want["circuit_evaluations"] == 601
        assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL
        assert abs(r.energy - want["energy"]) < E_TOL and r.energy == r.trajectory[-1]
        assert abs(r.theta[0] - want["theta"][0]) < TH_TOL


def test_run_vqe_tolerance_mode_iterations(gpu, ref):
    V = gpu
    H2 = V.AnsatzSpec.h2_double_excitation()
    cfg = V.AdamConfig(max_iterations=5000, gradient_tolerance=1e-8)
    for d in [0.7414, 1.2, 2.6]:  # test_vqe.cpp:152-169
        h = ref.build_h2_hamiltonian(d)
        want = ref.run_vqe(h, max_iter=5000, tol=1e-8)
        r = V.run_vqe(to_v(V, h), H2, cfg)
        assert r.iterations_run == want["iterations_run"]
        assert len(r.trajectory) == r.iterations_run + 1
        assert abs(r.energy - want["energy"]) < E_TOL
    r = V.run_vqe(to_v(V, ref.build_h2_hamiltonian(0.7414)), H2, V.AdamConfig(gradient_tolerance=1e3))
    assert r.iterations_run == 0 and len(r.trajectory) == 1 and r.circuit_evaluations == 3
    r = V.run_vqe(to_v(V, ref.build_h2_hamiltonian(0.9)), H2, V.AdamConfig(max_iterations=5))
    assert r.circuit_evaluations == 16


def test_run_vqe_errors_and_init(gpu, ref):
    V = gpu
    H2 = V.AnsatzSpec.h2_double_excitation()
    bad = V.QubitHamiltonian(4, [V.PauliTerm(complex(float("nan"), 0.0), [])])
    with pytest.raises(RuntimeError, match=r"non-finite energy at iteration 0; theta = 0\.000000"):
        V.run_vqe(bad, H2)
    h = to_v(V, ref.build_h2_hamiltonian(0.7414))
    with pytest.raises(ValueError, match="initial parameter count mismatch"):
        V.run_vqe(h, H2, V.AdamConfig(), [0.1, 0.2])
    r = V.run_vqe(h, H2, V.AdamConfig(max_iterations=0), [0.25])
    assert r.theta == [0.25] and abs(r.energy - V.energy([0.25], h, H2)) < E_TOL
    a = V.run_vqe(h, H2, V.AdamConfig(max_iterations=80))
    b = V.run_vqe(h, H2, V.AdamConfig(max_iterations=80))
    assert a.trajectory == b.trajectory and a.theta == b.theta  # test_vqe.cpp:216-226


@pytest.mark.parametrize("theta0", [2.0 ** 28 - 0.015, -(2.0 ** 28) + 0.015, 3.0e8, 1.0e12])
def test_run_vqe_h2_large_theta_trig_path(gpu, ref, theta0):
    """The H2 loop's short-range sincos hands over to the library sincos
    once |theta| >= 2^28 (fastmath.cuh): trajectories stay on the reference's,
    including a run that crosses the threshold mid-optimisation."""
    V = gpu
    H2 = V.AnsatzSpec.h2_double_excitation()
    h = ref.build_h2_hamiltonian(0.7414)
    want = ref.run_vqe(h, max_iter=40, init=[theta0])
    r = V.run_vqe(to_v(V, h), H2, V.AdamConfig(max_iterations=40), [theta0])
    assert r.iterations_run == want["iterations_run"] == 40
    assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL
    assert r.theta[0] == pytest.approx(want["theta"][0], rel=1e-15, abs=1e-9)


@pytest.mark.parametrize("key", ["tfim4", "zsum5", "tfim6", "tfim8"])
def test_run_vqe_hea_matches_golden(gpu, golden, key):
    V = gpu
    g = golden("vqe_runs.json")["hea"][key]
    n = g["hamiltonian"]["n_qubits"]
    h, _ = ham_from_text(V, n, g["hamiltonian"]["text"])
    r = V.run_vqe(h, V.AnsatzSpec.hardware_efficient(g["layers"]),
                  V.AdamConfig(learning_rate=g["lr"], max_iterations=g["max_iterations"]), [g["theta_init"]] * (2 * n))
    assert np.max(np.abs(np.array(r.trajectory) - g["trajectory"])) < E_TOL
    assert np.max(np.abs(np.array(r.theta) - g["theta"])) < 1e-9
    assert r.circuit_evaluations == g["circuit_evaluations"]


def test_run_vqe_batch(gpu, ref):
    V = gpu
    hs = [to_v(V, ref.build_h2_hamiltonian(d)) for d in [0.4, 0.8, 1.5, 2.9]]
    rs = V.run_vqe_batch(hs, V.AnsatzSpec.h2_double_excitation(), V.AdamConfig(max_iterations=50))
    for h, r in zip(hs, rs):
        one = V.run_vqe(h, V.AnsatzSpec.h2_double_excitation(), V.AdamConfig(max_iterations=50))
        assert r.trajectory == one.trajectory and r.theta == one.theta  # batch position independent


# ------------------------------------------------------------------ sweep
def test_run_sweep_default_matches_reference(gpu, golden):
    """The north-star workload: 100 bonds x 200 iterations."""
    V = gpu
    p = golden("pes_default.json")
    rep = V.run_sweep(V.SweepConfig(), trajectories=True)
    assert rep.all_ok
    assert [pt.bond_angstrom for pt in rep.points] == p["bond"]  # bitwise grid
    assert [pt.iterations for pt in rep.points] == p["iterations"]
    err = max(abs(pt.energy_hartree - e) for pt, e in zip(rep.points, p["energy"]))
    assert err < E_TOL, err
    assert max(abs(pt.theta_star[0] - t) for pt, t in zip(rep.points, p["theta"])) < TH_TOL
    i = int(np.argmin([pt.energy_hartree for pt in rep.points]))
    assert 0.70 <= rep.points[i].bond_angstrom <= 0.78 and abs(rep.points[i].energy_hartree + 1.137) < 0.005
    assert all(len(pt.trajectory) == 201 for pt in rep.points)


def test_run_sweep_tolerance_mode_iterations(gpu, golden):
    V = gpu
    t = golden("pes_default.json")["tol_mode"]
    rep = V.run_sweep(V.SweepConfig(adam=V.AdamConfig(max_iterations=5000, gradient_tolerance=1e-8)))
    assert [pt.iterations for pt in rep.points] == t["iterations"]  # bit-identical counts
    assert max(abs(pt.energy_hartree - e) for pt, e in zip(rep.points, t["energy"])) < E_TOL
    assert max(abs(pt.theta_star[0] - x) for pt, x in zip(rep.points, t["theta"])) < TH_TOL


def test_run_sweep_worker_and_chunk_independence(gpu):
    # test_sweep.cpp:101-129 / acceptance criterion 8
    V = gpu
    base = dict(d_min=0.5, d_max=2.0, n_points=8, adam=V.AdamConfig(max_iterations=25))
    reps = [V.run_sweep(V.SweepConfig(workers=w, **base)) for w in (1, 2, 3)]
    for rep in reps:
        assert rep.all_ok and len(rep.per_worker_seconds) >= 1
        for a, b in zip(rep.points, reps[0].points):
            assert (a.bond_angstrom, a.energy_hartree, a.theta_star, a.iterations) == \
                   (b.bond_angstrom, b.energy_hartree, b.theta_star, b.iterations)
    # rank-sharded (one process per GPU) slices reassemble the same points
    pts = []
    for r in range(3):
        pts += V.run_sweep(V.SweepConfig(chunk_index=r, n_chunks=3, **base)).points
    assert [(p.bond_angstrom, p.energy_hartree, p.iterations) for p in pts] == \
           [(p.bond_angstrom, p.energy_hartree, p.iterations) for p in reps[0].points]


def test_run_sweep_failing_point(gpu):
    # test_sweep.cpp:131-143
    V = gpu
    rep = V.run_sweep(V.SweepConfig(d_min=0.01, d_max=1.0, n_points=2, adam=V.AdamConfig(max_iterations=10)))
    assert not rep.all_ok and not rep.points[0].ok and rep.points[0].error
    assert "outside" in rep.points[0].error and math.isnan(rep.points[0].energy_hartree)
    assert rep.points[1].ok
    with pytest.raises(ValueError, match="workers must be >= 1"):
        V.run_sweep(V.SweepConfig(workers=0))


def test_scaling_study_zsum(gpu, golden):
    # test_sweep.cpp:195-212 configuration vs the reference's fixture
    V = gpu
    g = golden("scaling_zsum.json")
    c = g["config"]
    recs = V.run_scaling_study(V.ScalingConfig(qubits=c["qubits"], layers=c["layers"], iterations=c["iterations"],
                                               learning_rate=c["learning_rate"], z_sum_mode=True))
    for r, w in zip(recs, g["records"]):
        assert r["n_qubits"] == w["n_qubits"] and r["state_bytes"] == w["state_bytes"]
        assert r["iterations_run"] == w["iterations_run"]
        assert abs(r["final_energy"] - w["final_energy"]) < E_TOL
    with pytest.raises(ValueError, match="refusing 28 qubits"):
        V.run_scaling_study(V.ScalingConfig(qubits=[28]))
    with pytest.raises(ValueError, match=">= 2 qubits"):
        V.run_scaling_study(V.ScalingConfig(qubits=[1]))


def test_scaling_study_tfim_wide_matches_oracle(gpu, orc):
    """HBM engine path (n > 5) for run_scaling_study semantics."""
    V = gpu
    for n in [8, 12]:
        h = orc.build_tfim(n, 1.0, 1.0)
        want = orc.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=3, init=[0.1] * (2 * n))
        rec = V.run_scaling_study(V.ScalingConfig(qubits=[n], iterations=3))[0]
        assert abs(rec["final_energy"] - want["energy"]) < E_TOL and rec["iterations_run"] == 3


# ------------------------------------------- full-size property checks
def test_large_register_properties(gpu):
    """n = 28 (4 GiB fp64): oracle-free, size-independent properties:
    norm preserved, RY(a)RY(b) = RY(a+b) up to rounding, X X = I exactly,
    DE(t) DE(-t) = I, expectation of Z-sum on |0..0> = n."""
    V = gpu
    n = 28
    psi = V.StateVector(n)
    V.apply_circuit(psi, [V.Gate.ry(0.3, q) for q in range(n)])
    assert abs(psi.norm() - 1.0) < 1e-10
    e = V.expectation(psi, V.build_z_sum(n))
    assert abs(e - n * math.cos(0.3)) < 1e-9
    V.apply_circuit(psi, [V.Gate.pauli_x(0), V.Gate.pauli_x(0), V.Gate.cnot(3, 27), V.Gate.cnot(3, 27)])
    assert abs(V.expectation(psi, V.build_z_sum(n)) - e) < 1e-12
    V.apply_circuit(psi, [V.Gate.double_excitation(0.9, 0, 1, 2, 3), V.Gate.double_excitation(-0.9, 0, 1, 2, 3)])
    V.apply_circuit(psi, [V.Gate.ry(-0.3, q) for q in range(n)])
    z = V.expectation(psi, V.build_z_sum(n))
    assert abs(z - n) < 1e-9


# ------------------------------------------------------- adjoint gradient
@pytest.mark.parametrize("n", [4, 7, 10])
def test_adjoint_gradient_matches_parameter_shift_oracle(gpu, orc, n):
    """Adjoint (one forward + one backward sweep) vs the reference's
    parameter-shift rule (vqe.hpp:112-127) on the oracle."""
    V = gpu
    rng = np.random.default_rng(40 + n)
    hea = V.AnsatzSpec.hardware_efficient(2)
    for h in [orc.build_tfim(n, 1.0, 0.8), orc.canonicalize(random_hamiltonian(random.Random(n), n, 20))]:
        th = rng.uniform(-2, 2, 2 * n)
        g = V.gradient(th, to_v(V, h), hea, method="adjoint")
        assert np.max(np.abs(g - orc.gradient(1, 2, th, h))) < E_TOL
    h2 = orc.build_h2_hamiltonian(0.9)
    g = V.gradient([0.4], to_v(V, h2), V.AnsatzSpec.h2_double_excitation(), method="adjoint")
    assert abs(g[0] - orc.gradient(0, 0, [0.4], h2)[0]) < E_TOL


def test_adjoint_run_vqe_matches_golden(gpu, golden):
    V = gpu
    for key in ["tfim6", "tfim8"]:
        g = golden("vqe_runs.json")["hea"][key]
        n = g["hamiltonian"]["n_qubits"]
        h, _ = ham_from_text(V, n, g["hamiltonian"]["text"])
        r = V.run_vqe(h, V.AnsatzSpec.hardware_efficient(g["layers"]),
                      V.AdamConfig(learning_rate=g["lr"], max_iterations=g["max_iterations"]), [g["theta_init"]] * (2 * n),
                      method="adjoint")
        assert np.max(np.abs(np.array(r.trajectory) - g["trajectory"])) < E_TOL
        assert np.max(np.abs(np.array(r.theta) - g["theta"])) < 1e-9


def test_adjoint_equals_shift_at_width_20(gpu):
    """Both engines of ours at a width the oracle would take minutes on."""
    V = gpu
    n = 20
    h = V.build_tfim(n, 1.0, 1.0)
    th = np.random.default_rng(7).uniform(-1, 1, 2 * n)
    hea = V.AnsatzSpec.hardware_efficient(2)
    ga = V.gradient(th, h, hea, method="adjoint")
    gs = V.gradient(th, h, hea, method="shift")
    assert np.max(np.abs(ga - gs)) < 1e-10


def test_small_register_adjoint_runs_match_oracle(gpu, orc):
    """n <= 5 run_vqe with method="adjoint" takes the one-launch register
    engine; its trajectory still matches the reference's run_vqe."""
    V = gpu
    for n in [3, 4, 5]:
        h = orc.build_tfim(n, 1.0, 0.7)
        want = orc.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=5, init=[0.1] * (2 * n))
        for method in ("adjoint", "shift"):
            r = V.run_vqe(to_v(V, h), V.AnsatzSpec.hardware_efficient(2), V.AdamConfig(learning_rate=0.05, max_iterations=5),
                          [0.1] * (2 * n), method=method)
            assert abs(r.energy - want["energy"]) < E_TOL


def test_batched_shift_run_matches_adjoint_at_width_16(gpu):
    """Parameter shift at n = 16 runs the 2P + 1 circuits as one batch
    (padded full-height tile passes; the final energy evaluates one entry):
    same trajectory as the adjoint engine."""
    V = gpu
    n = 16
    h = V.build_tfim(n, 1.0, 1.0)
    hea = V.AnsatzSpec.hardware_efficient(2)
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=3)
    rs = V.run_vqe(h, hea, cfg, [0.1] * (2 * n), method="shift")
    ra = V.run_vqe(h, hea, cfg, [0.1] * (2 * n), method="adjoint")
    assert len(rs.trajectory) == len(ra.trajectory) == 4
    assert np.max(np.abs(np.array(rs.trajectory) - np.array(ra.trajectory))) < 1e-10
    assert np.max(np.abs(np.array(rs.theta) - np.array(ra.theta))) < 1e-10


@pytest.mark.parametrize("n", [12, 17])
def test_shared_prefix_shift_batch_is_bitwise(gpu, n, monkeypatch):
    """The batched parameter-shift family copies entry 0's state into each
    shifted entry before the first tile pass that uses its parameter; the
    energies and gradients are bitwise those of running every entry from
    |0..0> (VQF_NO_SHARED_PREFIX=1)."""
    V = gpu
    h = V.build_tfim(n, 1.0, 0.9)
    hea = V.AnsatzSpec.hardware_efficient(2)
    th = list(np.random.default_rng(n).uniform(-1.5, 1.5, 2 * n))
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=2)
    g1 = V.gradient(th, h, hea, method="shift")
    r1 = V.run_vqe(h, hea, cfg, th, method="shift")
    monkeypatch.setenv("VQF_NO_SHARED_PREFIX", "1")
    g0 = V.gradient(th, h, hea, method="shift")
    r0 = V.run_vqe(h, hea, cfg, th, method="shift")
    assert np.array_equal(np.asarray(g1), np.asarray(g0))
    assert r1.trajectory == r0.trajectory and list(r1.theta) == list(r0.theta)


def test_chunked_shift_batches_are_bitwise(gpu, monkeypatch):
    """A family larger than the memory budget runs in chunks (base + up to
    K - 1 shifted circuits each; VQF_SHIFT_MAX_BATCH caps K here): bitwise
    the energies of the one-circuit-at-a-time path."""
    V = gpu
    n = 12
    h = V.build_tfim(n, 1.0, 0.6)
    hea = V.AnsatzSpec.hardware_efficient(2)
    th = list(np.random.default_rng(3).uniform(-1.5, 1.5, 2 * n))
    monkeypatch.setenv("VQF_SHIFT_MAX_BATCH", "9")
    g_chunk = V.gradient(th, h, hea, method="shift")
    monkeypatch.setenv("VQF_SHIFT_MAX_BATCH", "1")
    g_seq = V.gradient(th, h, hea, method="shift")
    monkeypatch.delenv("VQF_SHIFT_MAX_BATCH")
    g_full = V.gradient(th, h, hea, method="shift")
    assert np.array_equal(np.asarray(g_chunk), np.asarray(g_seq))
    assert np.array_equal(np.asarray(g_full), np.asarray(g_seq))


def test_adjoint_large_hamiltonian_falls_back_and_checks_residue(gpu, orc):
    """Hamiltonians beyond the adjoint tables (> 256 flip groups) take the
    parameter-shift engine under method="adjoint" instead of failing; the
    adjoint path raises energy()'s imaginary-residue error like shift."""
    V = gpu
    n = 10
    h = orc.canonicalize(random_hamiltonian(random.Random(31), n, 400))
    th = np.random.default_rng(31).uniform(-1, 1, 2 * n)
    hea = V.AnsatzSpec.hardware_efficient(2)
    g = V.gradient(th, to_v(V, h), hea, method="adjoint")
    assert np.max(np.abs(g - orc.gradient(1, 2, th, h))) < E_TOL
    r = V.run_vqe(to_v(V, h), hea, V.AdamConfig(learning_rate=0.05, max_iterations=2), list(th), method="adjoint")
    want = orc.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=2, init=list(th))
    assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL
    bad = V.QubitHamiltonian(n, [V.PauliTerm(1.0, [(0, 1)]), V.PauliTerm(0.5j, [(3, 3)])])
    with pytest.raises(RuntimeError, match="imaginary residue"):
        V.gradient(th, bad, hea, method="adjoint")


def test_pes_kernel_device_hamiltonians_match_golden(gpu, golden):
    """The Hamiltonians the fused PES kernel builds on the device (HF + JW in
    the kernel prologue) against the reference's (tests/golden/
    h2_hamiltonians.json, from oracle/_ref's chem.hpp; goldens of
    test_chem.cpp:223-247) at 1e-12, and the HF summaries against
    run_hartree_fock."""
    V = gpu
    g = golden("h2_hamiltonians.json")
    keys = list(g["hamiltonians"])
    got = V.pes_device_hamiltonians([float(k) for k in keys])
    for b, (h, hf) in zip(keys, got):
        want, _ = ham_from_text(V, 4, g["hamiltonians"][b]["text"])
        wd = {tuple(t.axes): complex(t.coefficient).real for t in want.terms}
        gd = {tuple(t.axes): complex(t.coefficient).real for t in h.terms}
        assert set(gd) == set(wd), b
        assert max(abs(gd[k] - wd[k]) for k in wd) < 1e-12, b
        assert abs(hf["hf_energy"] - g["hartree_fock"][b]["hf_energy"]) < 1e-12
        assert hf["scf_iterations"] == g["hartree_fock"][b]["scf_iterations"]


# --------------------------------------------------- fp32 (complex64) path
F32_E_TOL = 1e-5  # north_star: energies within 1e-5 in fp32


@pytest.mark.parametrize("n", [4, 7, 12, 16, 20, 24])
def test_f32_energy_and_gradient_within_1e5(gpu, ref, n):
    """energy / gradient with complex64 states against the reference's fp64
    energy() (vqe.hpp:99-127) on TFIM and a random Pauli sum."""
    V = gpu
    hea = V.AnsatzSpec.hardware_efficient(2)
    th = np.random.default_rng(n).uniform(-1.5, 1.5, 2 * n)
    for h in [ref.build_tfim(n, 1.0, 0.9), ref.canonicalize(ref.random_hamiltonian(20260804, n, 32))]:
        e64 = ref.energy(1, 2, th, h)
        assert abs(V.energy(th, to_v(V, h), hea, dtype="f32") - e64) < F32_E_TOL
        if n <= 12:
            g64 = ref.gradient(1, 2, th, h)
            for method in ("shift", "adjoint"):
                g = V.gradient(th, to_v(V, h), hea, method=method, dtype="f32")
                assert np.max(np.abs(g - g64)) < F32_E_TOL, method


@pytest.mark.parametrize("n", [4, 10, 18])
def test_f32_run_vqe_fixed_iterations(gpu, ref, n):
    """run_vqe in fp32 (fixed iteration count) follows the reference's fp64
    trajectory within 1e-5; tol mode is refused (fp32 cannot reproduce the
    reference's stop decisions)."""
    V = gpu
    h = ref.build_tfim(n, 1.0, 1.0)
    want = ref.run_vqe(h, kind=1, layers=2, lr=0.05, max_iter=3, init=[0.1] * (2 * n))
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=3)
    for method in ("shift", "adjoint"):
        r = V.run_vqe(to_v(V, h), V.AnsatzSpec.hardware_efficient(2), cfg, [0.1] * (2 * n), method=method, dtype="f32")
        assert r.iterations_run == 3 and len(r.trajectory) == 4
        # complex64 amplitudes carry ~6e-8 relative rounding per gate, so
        # over an optimisation the bar is relative once |E| > 1
        bar = F32_E_TOL * np.maximum(1.0, np.abs(want["trajectory"]))
        assert np.all(np.abs(np.array(r.trajectory) - want["trajectory"]) < bar), method
        assert np.max(np.abs(np.array(r.theta) - want["theta"])) < 1e-4
    with pytest.raises(ValueError, match="fixed-iteration"):
        V.run_vqe(to_v(V, h), V.AnsatzSpec.hardware_efficient(2),
                  V.AdamConfig(max_iterations=5, gradient_tolerance=1e-3), dtype="f32")


def test_f32_scaling_study(gpu, ref):
    V = gpu
    recs = V.run_scaling_study(V.ScalingConfig(qubits=[6, 14], iterations=2, dtype="f32"))
    want = ref.run_scaling_study([6, 14], iterations=2)
    for r, w in zip(recs, want):
        assert r["state_bytes"] == (1 << r["n_qubits"]) * 8
        assert abs(r["final_energy"] - w["final_energy"]) < F32_E_TOL and r["iterations_run"] == 2


@pytest.mark.parametrize("n,dtype", [(11, "f64"), (14, "f64"), (20, "f64"), (12, "f32"), (17, "f32")])
def test_expectation_tile_passes_single_bit_flips(gpu, orc, n, dtype):
    """Single-bit flip groups (X_q / Y_q dressed with Z's, one or two terms
    per group) go through the gathered-tile multi-group passes
    (expect_tile.cu); every bit position, Y signs, complex phases and the
    tile-constant parity against the oracle."""
    V = gpu
    pr = random.Random(500 + n)
    terms = []
    for q in range(n):
        dress = sorted(pr.sample([w for w in range(n) if w != q], min(3, n - 1)))
        terms.append((pr.uniform(-2, 2), [(q, 1)]))                                     # X_q
        if q % 2 == 0:
            axes = sorted([(q, 2)] + [(w, 3) for w in dress])                          # Y_q Z...
            terms.append((pr.uniform(-2, 2), axes))
    terms += [(0.7, [(0, 3), (n - 1, 3)]), (-0.3, [])]
    h = orc.canonicalize(Ham(n, terms))
    psi0 = random_state(np.random.default_rng(n), n)
    psi = V.StateVector(n, dtype=dtype)
    psi.amplitudes = psi0
    got = V.expectation(psi, to_v(V, h))
    want = orc.expectation(n, psi0, h)
    assert abs(got - want) < (E_TOL if dtype == "f64" else 1e-5 * max(1.0, abs(want)))
    plan = V.expectation_plan(to_v(V, h))
    assert plan["state_passes"] < n  # groups share tile passes


@pytest.mark.parametrize("n,batch,n_diag", [(11, 1, 10), (14, 2, 32), (20, 1, 24), (22, 3, 45)])
def test_expectation_diagonal_folded_into_tile_pass(gpu, orc, n, batch, n_diag, monkeypatch):
    """fp64: a real diagonal group of <= 32 Z strings is evaluated inside one
    gathered-tile pass (Walsh-Hadamard over the register slots, tile signs
    by ballot) instead of its own pass; Z strings on every kind of bit
    (register slots, thread bits, tile bits), batched entries, against the
    oracle and against the unfolded plan (more than 32 strings: not folded)."""
    V = gpu
    pr = random.Random(900 + n)
    terms = [(pr.uniform(-2, 2), [(q, 1)]) for q in range(n)]  # single-bit flip groups -> tile passes
    for _ in range(n_diag):
        ws = sorted(pr.sample(range(n), pr.randint(1, 4)))
        terms.append((pr.uniform(-2, 2), [(w, 3) for w in ws]))
    h = orc.canonicalize(Ham(n, terms))
    n_z = sum(1 for _, axes in h.terms if axes and all(p == 3 for _, p in axes))
    hv = to_v(V, h)
    rng = np.random.default_rng(n + 5)
    psis = [random_state(rng, n) for _ in range(batch)]
    s = V.StateVector(n, batch=batch)
    s.amplitudes = np.concatenate(psis)
    folded = V.expectation_plan(hv)["state_passes"]
    got = np.atleast_1d(V.expectation(s, hv))
    for g, p in zip(got, psis):
        assert abs(g - orc.expectation(n, p, h)) < E_TOL
    monkeypatch.setenv("VQF_NO_DIAG_FOLD", "1")
    unfolded = V.expectation_plan(hv)["state_passes"]
    assert unfolded == folded + (1 if n_z <= 32 else 0)
    got2 = np.atleast_1d(V.expectation(s, hv))
    assert max(abs(a - b) for a, b in zip(got, got2)) < 1e-11


@pytest.mark.parametrize("n,batch,n_diag", [(12, 1, 20), (16, 2, 32), (21, 1, 28)])
def test_expectation_diagonal_folded_fp32(gpu, orc, n, batch, n_diag, monkeypatch):
    """fp32 (complex64) states fold the diagonal group into a gathered-tile
    pass too.  Z strings with distinct coefficients give several coefficient
    classes per register pattern (the overflow list), and a shared
    coefficient gives multi-string classes; against the fp64 oracle at the
    fp32 bar and against the unfolded fp32 plan (VQF_NO_DIAG_FOLD32)."""
    V = gpu
    pr = random.Random(1300 + n)
    terms = [(pr.uniform(-2, 2), [(q, 1)]) for q in range(n)]
    for i in range(n_diag):
        ws = sorted(pr.sample(range(n), pr.randint(1, 3)))
        c = -0.75 if i % 3 == 0 else pr.uniform(-2, 2)  # every third string shares one coefficient
        terms.append((c, [(w, 3) for w in ws]))
    h = orc.canonicalize(Ham(n, terms))
    hv = to_v(V, h)
    rng = np.random.default_rng(n + 11)
    psis = [random_state(rng, n) for _ in range(batch)]
    s = V.StateVector(n, batch=batch, dtype="f32")
    s.amplitudes = np.concatenate(psis)
    folded = V.expectation_plan(hv, "f32")["state_passes"]
    got = np.atleast_1d(V.expectation(s, hv))
    bar = 1e-5 * max(1.0, len(h.terms) / 10)
    for g, p in zip(got, psis):
        assert abs(g - orc.expectation(n, p, h)) < bar
    monkeypatch.setenv("VQF_NO_DIAG_FOLD32", "1")
    assert V.expectation_plan(hv, "f32")["state_passes"] == folded + 1
    got2 = np.atleast_1d(V.expectation(s, hv))
    assert max(abs(a - b) for a, b in zip(got, got2)) < bar
