"""B200-native rebuild of EngineCL's co-execution hot path (arXiv 1805.02755).

The product is native: ``_lib/libcoexec.so`` (C++ engine, schedulers,
metrics; include/ecl_engine.h) over ``_lib/libecl_cuda.so`` (CUDA device
layer and sm_100a kernels; include/ecl_cuda.h).  This package is the
Python mirror of the reference's coexec interface over that C-ABI.
"""
from . import coexec, workloads  # noqa: F401
from .coexec import *  # noqa: F401,F403
