"""B200-native DeFT-Flatten tree-attention decode (arXiv 2404.00242).

Drop-in for the reference's hot path (DecodingTree + PagePool +
partition_flatten + run_iteration) over hand-written sm_100a kernels reached
through the C ABI in include/treeattn_b200.h.
"""
from .api import IoStats, TreeAttention, run_iteration  # noqa: F401
from .capi import (CudaError, InvalidArgument, LogicError, NoDevice, OutOfMemory,  # noqa: F401
                   OutOfRange, TreeAttnError)

__all__ = ["TreeAttention", "run_iteration", "IoStats", "TreeAttnError", "InvalidArgument",
           "OutOfRange", "LogicError", "CudaError", "NoDevice", "OutOfMemory"]
