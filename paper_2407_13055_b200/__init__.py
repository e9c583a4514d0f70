"""ck32-b200: B200-native (sm_100a) 32-bit RNS-CKKS evaluation hot path.

Drop-in for the compute path of the reference C++ evaluator (ckks32): NTT /
INTT, base conversion inside ModUp / ModDown, KeyMult, HMult (+relinearize,
merged rescale), HRot, rescale and hoisted rotations, all as hand-written
CUDA kernels behind the C ABI in include/ck32_b200.h.  This package is the
Python mirror of that API (``ckks``) plus the reference wire formats
(``wire``).  There is no CPU fallback.
"""
from . import wire  # noqa: F401
from ._native import LIB_PATH, lib  # noqa: F401

__all__ = ["ckks", "wire", "lib", "LIB_PATH"]


def __getattr__(name):
    if name == "ckks":  # lazy: importing torch is slow on a cold box
        import importlib

        return importlib.import_module(__name__ + ".ckks")
    raise AttributeError(name)
