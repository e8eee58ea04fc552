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
rep = V.run_sweep(V.SweepConfig(n_points=4, adam=V.AdamConfig(max_iterations=10)))
print("ok", rep.all_ok)
