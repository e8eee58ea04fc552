"""GPU parity at the BASELINE config sizes, against the reference itself.

Config 3 (4-26 qubits, HEA + random Pauli sum / TFIM) at n = 20 and 24 and
config 4 (28-33 qubits, gate + expectation roofline) at n = 26 and 28, fp64
and fp32, through the C ABI, against oracle/_ref (the unmodified reference
headers, statevector.hpp:148-249, vqe.hpp:99-254, sweep.hpp:209-307) on the
reference's own seeded fixtures (tests/test_helpers.hpp:28-69: random_state
and random_hamiltonian from std::mt19937).  SingleExcitation, which the
reference lacks, is checked against the C restatement oracle (ORC_SE, pinned
to a dense embedding in tests/test_oracle.py).

Bars (BASELINE.json north_star; test_statevector.cpp:166): amplitudes 1e-12
and energies 1e-10 Ha in fp64, energies 1e-5 in fp32.  The reference's CPU
calls are single-threaded; independent ones run in a thread pool (ctypes
drops the GIL) so the suite stays within minutes.
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E_TOL = 1e-10
A_TOL = 1e-12
F32_E_TOL = 1e-5
HAM_SEED = 20260804      # mt19937(20260804), T = 32, real
STATE_SEED = 20260802    # test_statevector.cpp:150-166


def to_v(V, h):
    return V.QubitHamiltonian(h.n_qubits, [V.PauliTerm(c, a) for c, a in h.terms])


def upload(V, n, amps, dtype="f64"):
    psi = V.StateVector(n, dtype=dtype)
    psi.amplitudes = amps
    return psi


def every_wire_gates(n):
    """apply_gate on every wire (config 3): RY and X on each wire, the CNOT
    chain q -> q + 1 plus the wrap-around CNOT(n-1, 0), DoubleExcitation on
    the top, bottom and a straddling wire set."""
    g = [(1, 0.1 + 0.07 * q, [q]) for q in range(n)]
    g += [(0, 0.0, [q]) for q in range(0, n, 3)]
    g += [(2, 0.0, [q, q + 1]) for q in range(n - 1)] + [(2, 0.0, [n - 1, 0])]
    g += [(3, 0.8, [0, 1, 2, 3]), (3, -1.3, [n - 4, n - 3, n - 2, n - 1]), (3, 0.45, [n - 1, 1, n // 2, 3])]
    return g


def hea_gates(n, layers, theta):
    """vqe.hpp:81-93 hardware-efficient ansatz from |0...0>."""
    g, k = [], 0
    for _ in range(layers):
        for q in range(n):
            g.append((1, float(theta[k]), [q]))
            k += 1
        g += [(2, 0.0, [q, q + 1]) for q in range(n - 1)]
    return g


def gpu_gates(V, gates):
    return [V.Gate(k, a, tuple(w)) for k, a, w in gates]


# ------------------------------------------------------------- config 3
@pytest.mark.parametrize("n", [20, 24])
def test_config3_gates_on_every_wire(gpu, ref, n):
    """Fused circuit (tile passes) and one launch per gate, each against the
    reference's apply_gate sequence on its own random_state."""
    V = gpu
    psi0 = ref.random_state(STATE_SEED, n)
    gates = every_wire_gates(n)
    want = ref.apply_gates(n, psi0, gates)
    fused = upload(V, n, psi0)
    V.apply_circuit(fused, gpu_gates(V, gates))
    assert np.max(np.abs(fused.amplitudes - want)) < A_TOL
    per_gate = upload(V, n, psi0)
    for g in gpu_gates(V, gates):
        V.apply_gate(per_gate, g)
    assert np.max(np.abs(per_gate.amplitudes - want)) < A_TOL


@pytest.mark.parametrize("n", [20, 24])
def test_config3_expectation_tfim_and_random_sum(gpu, ref, n):
    V = gpu
    psi0 = ref.random_state(STATE_SEED + n, n)
    hams = [ref.build_tfim(n, 1.0, 1.0), ref.canonicalize(ref.random_hamiltonian(HAM_SEED, n, 32))]
    with ThreadPoolExecutor(len(hams)) as ex:
        want = list(ex.map(lambda h: ref.expectation(n, psi0, h), hams))
    psi = upload(V, n, psi0)
    psi32 = upload(V, n, psi0, "f32")
    for h, w in zip(hams, want):
        assert abs(V.expectation(psi, to_v(V, h)) - w) < E_TOL
        assert abs(V.expectation(psi32, to_v(V, h)) - w) < F32_E_TOL


def test_config3_hea_circuit_and_scaling_iteration_n20(gpu, ref):
    """One run_scaling_study iteration at n = 20 (HEA(2), theta0 = 0.1,
    lr 0.05; sweep.hpp:284-301) with TFIM, and one run_vqe iteration with the
    random 32-term sum, both gradient methods, against the reference's
    run_vqe (parameter shift)."""
    V = gpu
    n = 20
    tfim = ref.build_tfim(n, 1.0, 1.0)
    rnd = ref.canonicalize(ref.random_hamiltonian(HAM_SEED, n, 32))
    th = np.random.default_rng(5).uniform(-1.5, 1.5, 2 * n)
    with ThreadPoolExecutor(3) as ex:
        f_t = ex.submit(ref.run_vqe, tfim, kind=1, layers=2, lr=0.05, max_iter=1, init=[0.1] * (2 * n))
        f_r = ex.submit(ref.run_vqe, rnd, kind=1, layers=2, lr=0.05, max_iter=1, init=[0.1] * (2 * n))
        f_a = ex.submit(ref.prepare_ansatz, 1, 2, th, n)
        want_t, want_r, amps = f_t.result(), f_r.result(), f_a.result()
    # prepare_ansatz: fused HEA circuit
    assert np.max(np.abs(V.prepare_ansatz(V.AnsatzSpec.hardware_efficient(2), th, n).amplitudes - amps)) < A_TOL
    rec = V.run_scaling_study(V.ScalingConfig(qubits=[n], iterations=1))[0]
    assert rec["iterations_run"] == want_t["iterations_run"] == 1
    assert abs(rec["final_energy"] - want_t["energy"]) < E_TOL
    hea = V.AnsatzSpec.hardware_efficient(2)
    cfg = V.AdamConfig(learning_rate=0.05, max_iterations=1)
    for method in ("shift", "adjoint"):
        for h, want in ((tfim, want_t), (rnd, want_r)):
            r = V.run_vqe(to_v(V, h), hea, cfg, [0.1] * (2 * n), method=method)
            assert np.max(np.abs(np.array(r.trajectory) - want["trajectory"])) < E_TOL, method
            assert np.max(np.abs(np.array(r.theta) - want["theta"])) < 1e-9, method
            if method == "shift":  # the adjoint method counts forward circuits only
                assert r.circuit_evaluations == want["circuit_evaluations"]


def test_config3_energy_and_gradient_n24(gpu, ref):
    """n = 24: energy and three parameter-shift gradient components (first
    wire, middle, last parameter) against the reference's energy()."""
    V = gpu
    n = 24
    rnd = ref.canonicalize(ref.random_hamiltonian(HAM_SEED, n, 32))
    th = np.random.default_rng(24).uniform(-1.5, 1.5, 2 * n)
    ks = [0, n + n // 2, 2 * n - 1]
    jobs = [th] + [th + s * (math.pi / 2) * np.eye(2 * n)[k] for k in ks for s in (1, -1)]
    with ThreadPoolExecutor(len(jobs)) as ex:
        es = list(ex.map(lambda t: ref.energy(1, 2, t, rnd), jobs))
    hea = V.AnsatzSpec.hardware_efficient(2)
    h = to_v(V, rnd)
    assert abs(V.energy(th, h, hea) - es[0]) < E_TOL
    want = [0.5 * (es[1 + 2 * i] - es[2 + 2 * i]) for i in range(len(ks))]  # vqe.hpp:112-127
    for method in ("shift", "adjoint"):
        g = V.gradient(th, h, hea, method=method)
        assert max(abs(g[k] - w) for k, w in zip(ks, want)) < E_TOL, method


# ------------------------------------------------------------- config 4
def config4_gates(n):
    """RY on wires {0, n/2, n-1}, CNOT(q, q+1) at
    the top / middle, CNOT(n-2, n-1), CNOT(n-1, 0), DE(0..3), DE(n-4..n-1)."""
    m = n // 2
    return [(1, 0.3, [0]), (1, -0.7, [m]), (1, 1.1, [n - 1]), (2, 0.0, [0, 1]), (2, 0.0, [m, m + 1]),
            (2, 0.0, [n - 2, n - 1]), (2, 0.0, [n - 1, 0]), (3, 0.9, [0, 1, 2, 3]), (3, -0.4, [n - 4, n - 3, n - 2, n - 1])]


def se_gates(n):
    return [(4, 0.6, [0, n - 1]), (4, -1.2, [n // 2, n // 2 + 1]), (4, 0.35, [n - 2, 1])]


@pytest.mark.parametrize("n", [26, 28])
def test_config4_gates_fp64_and_fp32(gpu, ref, orc, n):
    """Each gate kind at its roofline positions on a seeded random state, fused
    and per gate, fp64 against the reference (SingleExcitation against the
    restatement oracle); fp32 from the same input within 1e-5 of the
    reference's expectation values."""
    V = gpu
    psi0 = ref.random_state(STATE_SEED, n)
    gates = config4_gates(n)
    ses = se_gates(n)
    want = ref.apply_gates(n, psi0, gates)
    want = orc.apply_gates(n, want, ses)
    fused = upload(V, n, psi0)
    V.apply_circuit(fused, gpu_gates(V, gates + ses))
    got = fused.amplitudes
    assert np.max(np.abs(got - want)) < A_TOL
    del got
    per_gate = upload(V, n, psi0)
    for g in gpu_gates(V, gates + ses):
        V.apply_gate(per_gate, g)
    assert np.max(np.abs(per_gate.amplitudes - want)) < A_TOL
    del per_gate
    h = ref.canonicalize(ref.random_hamiltonian(HAM_SEED, n, 8))
    e_want = ref.expectation(n, want, h)
    assert abs(V.expectation(fused, to_v(V, h)) - e_want) < E_TOL
    del fused
    f32 = upload(V, n, psi0, "f32")
    V.apply_circuit(f32, gpu_gates(V, gates + ses))
    assert abs(V.expectation(f32, to_v(V, h)) - e_want) < F32_E_TOL
    assert np.max(np.abs(f32.amplitudes - want)) < 1e-6


def test_config4_expectation_n26_fp64_fp32(gpu, ref):
    """TFIM (27 flip groups) and the random 32-term sum at n = 26."""
    V = gpu
    n = 26
    psi0 = ref.random_state(STATE_SEED + 1, n)
    hams = [ref.build_tfim(n, 1.0, 1.0), ref.canonicalize(ref.random_hamiltonian(HAM_SEED, n, 32))]
    with ThreadPoolExecutor(2) as ex:
        want = list(ex.map(lambda h: ref.expectation(n, psi0, h), hams))
    psi = upload(V, n, psi0)
    psi32 = upload(V, n, psi0, "f32")
    for h, w in zip(hams, want):
        assert abs(V.expectation(psi, to_v(V, h)) - w) < E_TOL
        assert abs(V.expectation(psi32, to_v(V, h)) - w) < F32_E_TOL


def test_config4_hea_layer_n28_fp64_fp32(gpu, ref):
    """One HEA layer (the fused tile passes the roofline bench times) at
    n = 28 from a random state, fp64 amplitudes vs the reference and fp32
    energies of a TFIM within 1e-5."""
    V = gpu
    n = 28
    psi0 = ref.random_state(STATE_SEED + 2, n)
    th = np.random.default_rng(28).uniform(-1.5, 1.5, n)
    gates = hea_gates(n, 1, th)
    want = ref.apply_gates(n, psi0, gates)
    psi = upload(V, n, psi0)
    V.apply_circuit(psi, gpu_gates(V, gates))
    assert np.max(np.abs(psi.amplitudes - want)) < A_TOL
    h = ref.build_z_sum(n)
    e_want = ref.expectation(n, want, h)
    assert abs(V.expectation(psi, to_v(V, h)) - e_want) < E_TOL
    del psi
    f32 = upload(V, n, psi0, "f32")
    V.apply_circuit(f32, gpu_gates(V, gates))
    assert abs(V.expectation(f32, to_v(V, h)) - e_want) < F32_E_TOL
