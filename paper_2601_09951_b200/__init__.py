"""B200-native VQE state-vector engine (drop-in for the VQE Forge hot path).

The product is ``libvqf_b200.so`` (CUDA, sm_100a) behind the C ABI in
``include/vqf_b200.h``; ``vqeforge`` mirrors the reference API on top of it.
"""
from . import vqeforge  # noqa: F401
from ._capi import LIB_PATH  # noqa: F401

__all__ = ["vqeforge", "LIB_PATH"]
