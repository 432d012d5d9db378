"""B200-native (sm_100a) drop-in for the hot path of the slab / GraphBLAS-HPCG reference:
the multigrid-preconditioned conjugate-gradient solve on the 27-point stencil.

The product is the CUDA shared library ``libslab_b200.so`` (hand-written kernels + the C ABI of
``include/slab_b200.h``). This package only locates/loads it and mirrors the reference's
operator API for Python callers; nothing here computes on the CPU.
"""
from ._capi import *  # noqa: F401,F403
from ._capi import LIB_PATH, SIGNATURES, load_library, launch_count, set_programmatic_launch, set_tuning  # noqa: F401
