"""ctypes binding of the C-ABI in include/abq_cuda.h (libabq_cuda.so).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2408_08554_b200/csrc``.  There is no fallback: if the library
is missing, importing the engine raises, and every compute entry point fails
with ABQ_ERR_CUDA when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# ABQ_LIB selects another build of the same library (tools: the trace build
# libabq_cuda_trace.so); the product path is the in-tree libabq_cuda.so
LIB_PATH = os.environ.get("ABQ_LIB") or os.path.join(_HERE, "libabq_cuda.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "abq_cuda.h")

ABQ_OK, ABQ_ERR_SHAPE, ABQ_ERR_VALUE, ABQ_ERR_OVERFLOW, ABQ_ERR_IO, ABQ_ERR_CUDA = range(6)
ABQ_ASYMMETRIC, ABQ_SYMMETRIC, ABQ_BALANCED = range(3)
ABQ_PER_TENSOR, ABQ_PER_CHANNEL, ABQ_PER_TOKEN = range(3)
ABQ_F16, ABQ_F64, ABQ_F32 = 0, 1, 2
ABQ_OUT_F16, ABQ_OUT_F64, ABQ_OUT_F32, ABQ_OUT_CORR_I64 = 0, 1, 2, 3
ABQ_GEMV_AUTO, ABQ_GEMV_POPC, ABQ_GEMV_RECOMB = 0, 1, 2


class QuantSpecC(C.Structure):
    _fields_ = [("bits", C.c_uint), ("scheme", C.c_int), ("granularity", C.c_int),
                ("alpha", C.c_double), ("beta", C.c_double)]


class TileConfigC(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("BM", "BN", "BK", "WM", "WN", "WK")]


class GemmStatsC(C.Structure):
    _fields_ = [("block_tiles", C.c_uint64), ("plane_pair_products", C.c_uint64)]


class QActC(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("scales", C.c_void_p), ("zero_points", C.c_void_p),
                ("rowsums", C.c_void_p), ("m", C.c_size_t), ("k", C.c_size_t), ("bits", C.c_uint)]


class WeightsC(C.Structure):
    _fields_ = [("planes", C.c_void_p), ("q", C.c_uint), ("n", C.c_size_t), ("k", C.c_size_t),
                ("scales", C.c_void_p), ("zero_points", C.c_void_p), ("colsums", C.c_void_p),
                ("per_tensor", C.c_int), ("frag", C.c_void_p), ("tc", C.c_void_p),
                ("next", C.c_void_p)]


class ActC(C.Structure):
    _fields_ = [("planes", C.c_void_p), ("p", C.c_uint), ("m", C.c_size_t), ("k", C.c_size_t),
                ("scales", C.c_void_p), ("zero_points", C.c_void_p), ("rowsums", C.c_void_p),
                ("per_tensor", C.c_int)]


_P = C.c_void_p
_S = C.c_size_t
_U = C.c_uint
_I = C.c_int

_SIGNATURES = {
    "abq_last_error": (C.c_char_p, []),
    "abq_version": (_I, []),
    "abq_launch_count": (C.c_uint64, []),
    "abq_fits_int32": (_I, [_U, _U, _S]),
    "abq_tile_valid": (_I, [C.POINTER(TileConfigC), _U, _U]),
    "abq_default_tile": (TileConfigC, [_U, _U]),
    "abq_padding_redundancy": (_I, [_S, _U, _S, C.POINTER(C.c_double)]),
    "abq_spec_levels": (_U, [C.POINTER(QuantSpecC)]),
    "abq_spec_planes": (_U, [C.POINTER(QuantSpecC)]),
    "abq_quantize": (_I, [_P, _I, _S, _S, C.POINTER(QuantSpecC), _P, _P, _P, _P, _P, _P]),
    "abq_quant_pack_act": (_I, [_P, _I, _S, _S, C.POINTER(QuantSpecC), _P, _P, _P, _P, _P, _P, _P]),
    "abq_bitpack": (_I, [_P, _S, _S, _U, _P, _P]),
    "abq_unpack": (_I, [_P, _U, _S, _S, _P, _P]),
    "abq_bmma": (_I, [_P, _U, _S, _U, _P, _U, _S, _U, _S, _P, _P]),
    "abq_gemm_btc": (_I, [_P, _U, _S, _S, _P, _U, _S, _S, _P, _P]),
    "abq_gemm_arbitrary": (_I, [_P, _U, _S, _S, _P, _U, _S, _S, C.POINTER(TileConfigC), _P,
                                C.POINTER(GemmStatsC), _P]),
    "abq_gemm_arbitrary_wide": (_I, [_P, _U, _S, _S, _P, _U, _S, _S, C.POINTER(TileConfigC), _P,
                                     C.POINTER(GemmStatsC), _P]),
    "abq_tile_engine_plan": (_I, [C.POINTER(TileConfigC), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "abq_gemm_naive": (_I, [_P, _U, _S, _S, _P, _U, _S, _S, _P, _P]),
    "abq_zero_point_correct_i32": (_I, [_P, _S, _S, _P, _P, _P, _P, _S, _P, _P]),
    "abq_zero_point_correct_i64": (_I, [_P, _S, _S, _P, _P, _P, _P, _S, _P, _P]),
    "abq_code_rowsums": (_I, [_P, _S, _S, _P, _P]),
    "abq_dequantize": (_I, [_P, _S, _S, _P, _P, _I, _P, _P]),
    "abq_plane_rowsums": (_I, [_P, _U, _S, _S, _P, _P]),
    "abq_weights_frag_bytes": (_S, [_U, _S, _S]),
    "abq_weights_prepack": (_I, [_P, _U, _S, _S, _P, _P]),
    "abq_weights_tc_bytes": (_S, [_U, _S, _S]),
    "abq_weights_prepack_tc": (_I, [_P, _U, _S, _S, _P, _P]),
    "abq_linear_planes": (_I, [C.POINTER(ActC), C.POINTER(WeightsC), _P, _I, _P]),
    "abq_linear_workspace_bytes": (_S, [_S, _S, _S, _U]),
    "abq_linear": (_I, [_P, _I, _S, _S, C.POINTER(QuantSpecC), C.POINTER(WeightsC), _P, _I, _P, _S,
                        _P, _P]),
    "abq_qact_codes_bytes": (_S, [_S, _S]),
    "abq_rmsnorm_quant": (_I, [_P, _P, C.c_float, _S, _S, C.POINTER(QuantSpecC), _P, C.POINTER(QActC), _P, _P]),
    "abq_silu_mul_quant": (_I, [_P, _P, _S, _S, C.POINTER(QuantSpecC), _P, C.POINTER(QActC), _P, _P]),
    "abq_stage_in": (_I, [_P, _P, _S, _P]),
    "abq_linear_host": (_I, [_P, _I, _S, _S, _P, C.POINTER(QuantSpecC), C.POINTER(WeightsC), _P, _I, _P, _S,
                             _P, _P]),
    "abq_linear_qact": (_I, [C.POINTER(QActC), C.POINTER(WeightsC), _P, _I, _P]),
    "abq_set_gemv_variant": (_I, [_I]),
    "abq_get_gemv_variant": (_I, []),
    "abq_set_gemm_schedule": (_I, [_I]),
    "abq_get_gemm_schedule": (_I, []),
    "abq_set_trace_buffer": (_I, [_P]),
    "abq_set_tuning": (_I, [C.c_char_p, C.c_longlong]),
}


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Every function name declared in include/abq_cuda.h."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(abq_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"libabq_cuda.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
