import sys; sys.path.insert(0, "/root/repo")
from paper_2601_09951_b200 import vqeforge as V
V.init(0)
h = V.build_h2_hamiltonian(0.7414)
H2 = V.AnsatzSpec.h2_double_excitation()
for mi, tol in [(200, None), (5000, None), (1000, None), (3000, None), (200, 1e-8), (5000, 1e-8), (2500, None), (2000, None)]:
    r = V.run_vqe(h, H2, V.AdamConfig(max_iterations=mi, gradient_tolerance=tol))
    print(mi, tol, r.iterations_run, r.trajectory[:3], r.energy, flush=True)
