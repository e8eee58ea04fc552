"""Max |d theta*| and |d E| of the default PES (fixed 200 and tol mode)
against the reference fixture (tests/golden/pes_default.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_09951_b200 import vqeforge as V  # noqa: E402

g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "pes_default.json")))
V.init(0)
rep = V.run_sweep(V.SweepConfig())
dth = max(abs(p.theta_star[0] - t) for p, t in zip(rep.points, g["theta"]))
de = max(abs(p.energy_hartree - e) for p, e in zip(rep.points, g["energy"]))
nbit = sum(p.theta_star[0] == t for p, t in zip(rep.points, g["theta"]))
print(f"fixed-200: max|dtheta*| = {dth:.3e}  max|dE| = {de:.3e}  bitwise theta* {nbit}/100")
t = g["tol_mode"]
rep = V.run_sweep(V.SweepConfig(adam=V.AdamConfig(max_iterations=5000, gradient_tolerance=1e-8)))
print("tol keys", list(t.keys()))
de = max(abs(p.energy_hartree - e) for p, e in zip(rep.points, t["energy"]))
same = [p.iterations for p in rep.points] == t["iterations"]
msg = f"tol-mode: max|dE| = {de:.3e} iterations identical: {same}"
if "theta" in t:
    msg += f" max|dtheta*| = {max(abs(p.theta_star[0] - x) for p, x in zip(rep.points, t['theta'])):.3e}"
print(msg)
