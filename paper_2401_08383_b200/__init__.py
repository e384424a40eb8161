"""B200-native ExFlow context-coherent expert-parallel MoE inference layer.

The hot path is hand-written sm_100a CUDA behind the C-ABI in
include/exflow_c.h (libexflow_b200.so). This package is the Python host
mirror of the reference's exflow:: surface used by tests and the bench.
"""
from . import _capi  # noqa: F401
from ._capi import (ExflowCommError, ExflowCudaError, ExflowError,  # noqa: F401
                    ExflowInvalidArgument)
from .build import build_library  # noqa: F401

__all__ = ["build_library", "ExflowError", "ExflowInvalidArgument", "ExflowCudaError",
           "ExflowCommError"]
