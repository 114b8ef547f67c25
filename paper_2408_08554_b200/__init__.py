"""paper_2408_08554_b200 -- B200-native (sm_100a) arbitrary-bit bit-plane
quantized matmul engine with the ABQ-LLM reference operator API.

The compute lives in libabq_cuda.so (paper_2408_08554_b200/csrc, C-ABI in
include/abq_cuda.h).  This package is the host-side mirror of the reference
interface used by the tests and the benchmark; the C++ mirror is include/abq/.
"""
from . import _lib  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import (BitPlaneMatrix, Error, GemmStats, IoError, Linear, OverflowError,  # noqa: F401
                  PackedWeights, QuantizedTensor, QuantSpec, ShapeError, TileConfig, ValueError,
                  bitpack, bmma, code_rowsums, default_tile, dequantize, fits_int32, gemm_arbitrary, gemm_btc,
                  gemm_arbitrary_wide, gemm_naive, linear_planes, padding_redundancy, plane_rowsums,
                  quantize, quantize_balanced, quantized_linear, unpack, zero_point_correct)
from . import io, model  # noqa: F401,E402  (weight files; toy block)
