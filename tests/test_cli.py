"""The reference-compatible CLI (tools/vqeforge_b200.cpp -> bin/vqeforge):
same subcommands, flags, output files and exit codes as the reference's
tools/vqeforge.cpp, checked against the golden fixtures made from the
reference itself (tests/golden/make_golden.py).  CPU tests use only the
host-side subcommands (exact, dump-hamiltonian, --version, usage errors);
the GPU tests run pes / bench / scaling on the B200 engine."""
from __future__ import annotations

import csv
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2601_09951_b200", "bin", "vqeforge")


def run(*args, cwd=None, timeout=600):
    if not os.path.exists(CLI):
        pytest.fail("bin/vqeforge not built (run __graft_entry__.build())")
    return subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=timeout)


def parse_text(text):
    """to_text lines -> [(coeff, pauli string)] (sparse_hamiltonian.hpp to_text)."""
    out = []
    for line in text.strip().splitlines():
        parts = line.split()
        out.append((float(parts[0]), float(parts[1]), " ".join(parts[2:])))
    return out


def test_version():
    r = run("--version")
    assert r.returncode == 0 and r.stdout.strip() == "0.1.0"


@pytest.mark.parametrize("form", ["sub", "sub_eq", "top"])
def test_dump_hamiltonian_matches_reference_text(golden, form):
    hams = golden("h2_hamiltonians.json")["hamiltonians"]
    for bond, rec in hams.items():
        if form == "sub":
            r = run("dump-hamiltonian", "--bond", bond)
        elif form == "sub_eq":
            r = run("dump-hamiltonian", f"--bond={bond}")
        else:
            r = run("--dump-hamiltonian", bond)
        assert r.returncode == 0, r.stderr
        got, want = parse_text(r.stdout), parse_text(rec["text"])
        assert [g[2] for g in got] == [w[2] for w in want]  # same terms, same canonical order
        for g, w in zip(got, want):
            assert abs(g[0] - w[0]) <= 1e-13 and g[1] == w[1] == 0.0


def test_exact_matches_reference(golden):
    for bond, e in golden("h2_hamiltonians.json")["exact_ground_energy"].items():
        r = run("exact", "--bond", bond)
        assert r.returncode == 0, r.stderr
        assert r.stdout == "%.6f\n" % e


@pytest.mark.parametrize(
    "args,needle",
    [
        ((), "usage"),
        (("frobnicate",), "unknown subcommand"),
        (("pes", "--bogus", "1"), "unknown option"),
        (("pes", "--points"), "requires a value"),
        (("pes", "--points", "ten"), "not an integer"),
        (("exact",), "--bond is required"),
        (("exact", "--bond", "0.01"), "error: bond length"),
        (("exact", "--bond", "11"), "error: bond length"),
        (("bench", "--worker-list", "1,0"), "'0' is not a positive integer"),
        (("bench", "--worker-list", ""), "empty list"),
        (("scaling", "--qubits", "4,x"), "'x' is not a positive integer"),
        (("scaling", "--gradient", "finite-diff"), "expected shift or adjoint"),
    ],
)
def test_usage_errors_exit_2(args, needle):
    r = run(*args)
    assert r.returncode == 2
    assert needle in r.stderr


# ------------------------------------------------------------------ GPU
def _read_json(path):
    with open(path) as f:
        return json.load(f)


@pytest.mark.gpu
def test_pes_default_matches_golden(gpu, golden, tmp_path):
    g = golden("pes_default.json")
    r = run("pes", "--out-dir", str(tmp_path))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("equilibrium estimate: d = ")
    doc = _read_json(tmp_path / "pes.json")
    man = doc["manifest"]
    assert man["command"] == "pes" and man["version"] == "0.1.0"
    assert man["config"]["points"] == 100 and man["config"]["tolerance"] is None
    pts = doc["data"]["points"]
    assert doc["data"]["all_ok"] is True and len(pts) == 100
    assert [p["bond_angstrom"] for p in pts] == g["bond"]  # bitwise grid
    assert [p["iterations"] for p in pts] == g["iterations"]
    assert max(abs(p["energy_hartree"] - e) for p, e in zip(pts, g["energy"])) < 1e-10
    assert max(abs(p["theta_star"][0] - t) for p, t in zip(pts, g["theta"])) < 1e-12
    with open(tmp_path / "pes.csv") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["bond_angstrom", "energy_hartree", "theta_star", "iterations", "wall_seconds"]
    assert len(rows) == 101
    for row, e, it in zip(rows[1:], g["energy"], g["iterations"]):
        assert abs(float(row[1]) - e) <= 1e-11 * max(1.0, abs(e)) and int(row[3]) == it
    # argmin line: same as the golden grid argmin
    k = min(range(100), key=lambda i: g["energy"][i])
    assert "d = %.6f angstrom, E = %.6f hartree" % (g["bond"][k], g["energy"][k]) in r.stdout


@pytest.mark.gpu
def test_pes_tolerance_mode_matches_golden(gpu, golden, tmp_path):
    g = golden("pes_default.json")["tol_mode"]
    r = run("pes", "--tol", str(g["gradient_tolerance"]), "--iterations", str(g["max_iterations"]),
            "--workers", "2", "--out-dir", str(tmp_path))
    assert r.returncode == 0, r.stderr
    pts = _read_json(tmp_path / "pes.json")["data"]["points"]
    assert [p["iterations"] for p in pts] == g["iterations"]
    assert max(abs(p["energy_hartree"] - e) for p, e in zip(pts, g["energy"])) < 1e-10


@pytest.mark.gpu
def test_bench_writes_rows(gpu, tmp_path):
    r = run("bench", "--worker-list", "2,4", "--points", "20", "--iterations", "50", "--out-dir", str(tmp_path))
    assert r.returncode == 0, r.stderr
    doc = _read_json(tmp_path / "bench.json")
    rows = doc["data"]["rows"]
    assert rows[0]["workers"] == 1 and rows[0]["speedup_vs_w1"] == 1.0
    assert [x["workers"] for x in rows] == doc["manifest"]["config"]["worker_list"]
    assert all(x["total_seconds"] > 0 for x in rows)
    assert r.stdout.count("workers=") == len(rows)
    with open(tmp_path / "bench.csv") as f:
        assert f.readline().strip() == "workers,total_seconds,speedup_vs_w1,efficiency,amdahl_speedup"


@pytest.mark.gpu
@pytest.mark.parametrize("gradient", ["shift", "adjoint"])
def test_scaling_matches_golden(gpu, golden, tmp_path, gradient):
    g = golden("scaling_zsum.json")
    c = g["config"]
    r = run("scaling", "--qubits", ",".join(map(str, c["qubits"])), "--layers", str(c["layers"]),
            "--iterations", str(c["iterations"]), "--lr", str(c["learning_rate"]), "--z-sum",
            "--theta-init", str(c["theta_init"]), "--gradient", gradient, "--out-dir", str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = _read_json(tmp_path / "scaling.json")["data"]["rows"]
    for got, want in zip(rows, g["records"]):
        assert got["n_qubits"] == want["n_qubits"] and got["state_bytes"] == want["state_bytes"]
        assert got["iterations_run"] == want["iterations_run"]
        assert abs(got["final_energy"] - want["final_energy"]) < 1e-9
