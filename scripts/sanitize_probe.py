"""Small workloads of the round-2 kernels for compute-sanitizer: the
shared-memory engine (teams, grid, global-state), the distributed state
(virtual ranks), fused tiles and the gathered-tile expectation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V
from paper_2601_09951_b200.dsv import DistributedStateVector

V.init(0)
for n in (4, 6, 9, 14):
    V.run_scaling_study(V.ScalingConfig(qubits=[n], iterations=2))
V.run_scaling_study(V.ScalingConfig(qubits=[10], iterations=2, dtype="f32"))
d = DistributedStateVector(12, 4)
d.apply_circuit([(1, 0.1 * (q + 1), [q]) for q in range(12)] + [(2, 0.0, [q, q + 1]) for q in range(11)])
print(d.expectation(V.build_tfim(12, 1.0, 1.0)))
psi = V.StateVector(16)
V.apply_circuit(psi, [V.Gate.ry(0.1 * (q + 1), q) for q in range(16)] + [V.Gate.cnot(q, q + 1) for q in range(15)])
print(V.expectation(psi, V.build_tfim(16, 1.0, 1.0)))
print(V.run_vqe(V.build_tfim(16, 1.0, 1.0), V.AnsatzSpec.hardware_efficient(1), V.AdamConfig(max_iterations=1),
                method="adjoint").energy)
# fp32 fused tiles and expectation with the folded diagonal; a diagonal group
# with several coefficient classes per register pattern (overflow list)
psi32 = V.StateVector(16, dtype="f32")
V.apply_circuit(psi32, [V.Gate.ry(0.1 * (q + 1), q) for q in range(16)] + [V.Gate.cnot(q, q + 1) for q in range(15)])
print(V.expectation(psi32, V.build_tfim(16, 1.0, 1.0)))
terms = [V.PauliTerm(0.3 + 0.01 * q, [(q, 1)]) for q in range(16)]
terms += [V.PauliTerm(0.5 + 0.1 * q, [(q, 3), ((q + 1) % 16, 3)]) for q in range(16)]
terms += [V.PauliTerm(-0.7 - 0.05 * q, [(q, 3)]) for q in range(16)]
hmix = V.QubitHamiltonian(16, terms)
print(V.expectation(psi, hmix), V.expectation(psi32, hmix))
rep = V.run_sweep(V.SweepConfig(n_points=4, adam=V.AdamConfig(max_iterations=10)))
print("ok", rep.all_ok)
