"""The reference acceptance program's hot-path criteria
(tests/acceptance/acceptance_main.cpp:134-220, 431-446) run against the
engine: converged-sweep accuracy, the variational bound, shift rule vs
finite differences and mean-field consistency.  Same thresholds as the
reference; the random draws are our own (numpy MT19937), the criteria are
properties, not fixtures."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def to_v(V, h):
    return V.QubitHamiltonian(h.n_qubits, [V.PauliTerm(c, a) for c, a in h.terms])


def test_criterion_converged_sweep_accuracy(gpu, ref):
    """acceptance_main.cpp:134-153: all 100 grid points of a tol-mode sweep
    (1e-8, <= 5000 iterations) within 1e-6 Ha of the exact ground energy."""
    V = gpu
    rep = V.run_sweep(V.SweepConfig(adam=V.AdamConfig(max_iterations=5000, gradient_tolerance=1e-8)))
    assert rep.all_ok
    worst = 0.0
    for pt in rep.points:
        e0 = ref.exact_ground_energy(ref.build_h2_hamiltonian(pt.bond_angstrom))
        worst = max(worst, abs(pt.energy_hartree - e0))
    assert worst < 1e-6, worst


def test_criterion_variational_bound(gpu, ref):
    """acceptance_main.cpp:155-179: 10 bonds x 100 random angles never
    undercut the exact ground energy by more than 1e-10."""
    V = gpu
    rng = np.random.RandomState(402653189)
    spec = V.AnsatzSpec.h2_double_excitation()
    for _ in range(10):
        d = rng.uniform(0.3, 3.0)
        h = ref.build_h2_hamiltonian(d)
        e0 = ref.exact_ground_energy(h)
        hv = to_v(V, h)
        for th in rng.uniform(-np.pi, np.pi, 100):
            assert V.energy([th], hv, spec) >= e0 - 1e-10


def test_criterion_gradient_agreement(gpu, ref):
    """acceptance_main.cpp:181-206: the parameter-shift gradient matches
    central finite differences (step 1e-5) within 1e-7 at 100 random points."""
    V = gpu
    rng = np.random.RandomState(805306457)
    spec = V.AnsatzSpec.h2_double_excitation()
    step = 1e-5
    for _ in range(100):
        d, th = rng.uniform(0.3, 3.0), rng.uniform(-np.pi, np.pi)
        hv = to_v(V, ref.build_h2_hamiltonian(d))
        ps = V.gradient([th], hv, spec)[0]
        fd = (V.energy([th + step], hv, spec) - V.energy([th - step], hv, spec)) / (2 * step)
        assert abs(ps - fd) < 1e-7, (d, th, ps, fd)


def test_criterion_mean_field_consistency(gpu, ref):
    """acceptance_main.cpp:208-220: <HF|H|HF> equals the Hartree-Fock energy
    within 1e-8 on a 20-point grid (basis_state |1100> on the device)."""
    V = gpu
    for d in ref.bond_grid(0.3, 3.0, 20):
        h = ref.build_h2_hamiltonian(float(d))
        psi = V.basis_state(4, [1, 1, 0, 0])
        hf = ref.hartree_fock(float(d))
        assert abs(V.expectation(psi, to_v(V, h)) - hf["hf_energy"]) < 1e-8
