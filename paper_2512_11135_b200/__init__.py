"""paper_2512_11135_b200 -- B200-native (sm_100a) CKKS linear-transform hot path.

The product is the CUDA library libhx_b200.so (C-ABI, include/hx_b200.h) and the
helix C++ host library (include/helix/) above it; this Python package only
locates and binds the built shared libraries (hx.py) for tests and benchmarks.
"""
from .hx import Context, HxError, LIB_PATH, lib  # noqa: F401

__all__ = ["Context", "HxError", "LIB_PATH", "lib"]
