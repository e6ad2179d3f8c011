"""B200-native (sm_100a, fp64) Newton-Krylov-Schwarz time step of arXiv 2209.08001.

The product is the C-ABI library ``lib/libnks.so`` (include/nks.h); ``nks.py`` is its thin
ctypes binding.  There is no CPU fallback: without the built library or a CUDA device the
binding raises.
"""
from .nks import (PC_AS_BILU0, PC_NONE, PC_RAS_BILU0, PC_RRAS_BILU0, PC_RAS_SPECTRAL, PC_SPECTRAL, Grid, NKSError, Params, Solver, StepInfo,  # noqa: F401
                  decompose, load_library, make_grid, make_params, unique_id, version)
