"""The C++ drop-in header (include/vqeforge_b200/vqeforge.hpp) compiles with
g++ against libvqf_b200.so and passes reference-style checks
(tests/cpp/test_dropin.cpp).  CPU: compile + host-only subset; GPU: all."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2601_09951_b200")


@pytest.fixture(scope="module")
def dropin_binary(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cpp") / "test_dropin")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L", LIBDIR, "-lvqf_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_dropin_header_host_subset(dropin_binary):
    r = subprocess.run([dropin_binary, "--host-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("ok ")


@pytest.mark.gpu
def test_dropin_header_on_gpu(dropin_binary):
    r = subprocess.run([dropin_binary], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    assert r.stdout.startswith("ok ")


def test_block_engine_frame_compilation():
    """compile_block_program (csrc/vqe_block.cu) replayed on the host: the
    frame-tracked rotation passes and rewritten Pauli masks give the same
    energies as the direct HEA circuit + reference expectation formula
    (tests/cpp/block_frame_check.cpp), n = 4..15, 1-3 layers, fp64/fp32 plans."""
    exe = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"block_frame_check_{os.getpid()}")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(ROOT, "paper_2601_09951_b200", "csrc"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "block_frame_check.cpp"), "-L", LIBDIR, "-lvqf_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    try:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
        assert r.stdout.startswith("ok ")
    finally:
        os.unlink(exe)
