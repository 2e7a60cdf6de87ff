"""B200-native DADE distance-comparison hot path (arXiv 2411.17229).

The search path (rotation, coarse ranking, probe grouping, dimension-
progressive DCO scan, top-K merge) runs in libdade_gpu.so (sm_100a CUDA);
this package is the Python mirror of the reference's search API over its
C ABI (include/dade_gpu.h). Importing it without the built library raises.
"""
from ._capi import ConfigError, CudaError, DadeError, InvalidInput  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import evaluate_batch, partial_sums  # noqa: F401

__version__ = "0.1.0"
