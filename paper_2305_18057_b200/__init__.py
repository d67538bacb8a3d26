"""B200-native structured-grid finite-volume hot path of SENSEI (arXiv 2305.18057).

The product is libsfv.so (C ABI in include/sfv.h, CUDA kernels for sm_100a in
csrc/); `sfv` is its ctypes binding and `inputs` the seeded input generators.
"""
from . import inputs  # noqa: F401

__all__ = ["inputs", "sfv", "build"]
