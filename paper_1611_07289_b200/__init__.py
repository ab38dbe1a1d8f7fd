"""PVR (arXiv 1611.07289) super-resolution iteration, B200-native.

The product is libpvr.so (include/pvr.h): hand-written sm_100a CUDA kernels behind a
C ABI. This package holds its sources (csrc/), the in-tree build (build.py) and a thin
ctypes binding (pvr.py) with the same names as the C calls.
"""
from .pvr import (Context, PvrError, load_problem, pvr_plan_shards, pvr_version,  # noqa: F401
                  lib, SO_PATH)
from .pipeline import reconstruct  # noqa: F401
