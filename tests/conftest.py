"""Shared fixtures.  Markers: `gpu` = needs a B200 (run with -m gpu on the
GPU box); everything else runs on CPU in the build container."""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import load_orc

    return load_orc()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import load_ref

    r = load_ref()
    if r is None:
        pytest.skip("oracle/_ref/libvqf_ref.so not built")
    return r


@pytest.fixture(scope="session")
def V():
    from paper_2601_09951_b200 import vqeforge

    return vqeforge


@pytest.fixture(scope="session")
def gpu(V):
    """The CUDA engine on device 0.  Fails (does not skip) without a GPU:
    a GPU test that silently passes without the native path proves nothing."""
    n = V.device_count()
    if n < 1:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")
    V.init(0)
    return V


@pytest.fixture(scope="session")
def golden():
    def load(name):
        with open(os.path.join(GOLDEN, name)) as f:
            return json.load(f)

    return load
