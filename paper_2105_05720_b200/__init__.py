"""B200-native backend for the CoCoNet (arXiv 2105.05720) fused
compute/communication hot path.

The C-ABI library (libcoconet_cuda.so, include/coconet_cuda.h) holds the sm_100a
kernels; this package is its Python side (context, symmetric buffers, the fused
collectives, the torch optimizer integration) and the binding of GpuEngine,
the C++ drop-in for the reference's ccopt::Engine.
"""
from ._lib import (ALGO_AUTO, ALGO_ONE_SHOT, ALGO_TWO_SHOT, BF16, F16, F32, MATH_EXACT, MATH_FAST,
                   MAX, MIN, SUM, CoconetError)

__all__ = ["ALGO_AUTO", "ALGO_ONE_SHOT", "ALGO_TWO_SHOT", "BF16", "F16", "F32", "MATH_EXACT",
           "MATH_FAST", "MAX", "MIN", "SUM", "CoconetError"]
