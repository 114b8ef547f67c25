"""numpy/ctypes front-end of the CHECKER.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg -- never by the product
package.  Two back-ends with identical signatures:

  ``C``    liboracle.so   -- the C restatement (oracle/abq_oracle.c)
  ``REF``  _ref/libabqref.so -- the unmodified reference headers (ref_shim.cpp);
                              present where /root/reference was available at
                              build time (it travels to the GPU box prebuilt).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libabqref.so")

_P = C.c_void_p
_S = C.c_size_t
_U = C.c_uint
_I = C.c_int


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "all" if os.path.isdir("/root/reference/proj/include")
                    else os.path.join(HERE, "liboracle.so")], check=True)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def wpr(cols: int) -> int:
    return (cols + 63) // 64


class COracle:
    """oracle/abq_oracle.c"""

    def __init__(self, path: str = C_LIB_PATH):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_quantize.argtypes = [_P, _S, _S, _U, _I, _I, C.c_double, C.c_double, _P, _P, _P, _P, _P, _P]
        L.orc_bitpack.argtypes = [_P, _S, _S, _U, _P, _P]
        L.orc_unpack.argtypes = [_P, _U, _S, _S, _P]
        L.orc_bmma.argtypes = [_P, _U, _S, _U, _P, _U, _S, _U, _S, _P]
        L.orc_gemm_planes.argtypes = [_P, _U, _S, _P, _U, _S, _S, _P]
        L.orc_gemm_arbitrary_i32.argtypes = [_P, _U, _S, _P, _U, _S, _S, _P]
        L.orc_code_rowsums.argtypes = [_P, _S, _S, _P]
        L.orc_zero_point_correct.argtypes = [_P, _S, _S, _P, _P, _P, _P, _S, _P]
        L.orc_quantized_linear.argtypes = [_P, _S, _U, _P, _P, _I, _P, _S, _U, _P, _P, _I, _S, _P]
        L.orc_padding_redundancy.restype = C.c_double
        L.orc_padding_redundancy.argtypes = [_S, _U, _S]
        L.orc_fits_int32.argtypes = [_U, _U, _S]
        L.orc_tile_valid.argtypes = [_S, _S, _S, _S, _S, _S, _U, _U]
        L.orc_levels.argtypes = [_U, _I]
        L.orc_planes.argtypes = [_U, _I]
        L.orc_gemm_stats.argtypes = [_S, _S, _S, _S, _U, _U, _P, _P]
        L.orc_dequantize.argtypes = [_P, _S, _S, _I, _P, _P, _P]

    # quantizer.hpp:146-213
    def quantize(self, x, bits, scheme=0, granularity=0, alpha=1.0, beta=1.0, comp=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows, cols = x.shape
        groups = 1 if granularity == 0 else rows
        codes = np.zeros((rows, cols), np.uint8)
        scales = np.zeros(groups, np.float64)
        zps = np.zeros(groups, np.int32)
        bad = np.zeros(1, np.int64)
        ca = cb = None
        if comp is not None:
            ca = np.ascontiguousarray(comp[0], dtype=np.float64)
            cb = np.ascontiguousarray(comp[1], dtype=np.float64)
        st = self.lib.orc_quantize(_p(x), rows, cols, bits, scheme, granularity, alpha, beta, _p(ca),
                                   _p(cb), _p(codes), _p(scales), _p(zps), _p(bad))
        if st:
            raise ValueError(f"oracle quantize status {st} (bad index {int(bad[0])})")
        return codes, scales, zps

    def bitpack(self, codes, bits):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        rows, cols = codes.shape
        out = np.zeros((bits, rows, wpr(cols)), np.uint64)
        bad = np.zeros(1, np.int64)
        st = self.lib.orc_bitpack(_p(codes), rows, cols, bits, _p(out), _p(bad))
        if st:
            raise ValueError(f"oracle bitpack: code out of range at flat index {int(bad[0])}")
        return out

    def unpack(self, planes, cols):
        planes = np.ascontiguousarray(planes, dtype=np.uint64)
        bits, rows, _ = planes.shape
        out = np.zeros((rows, cols), np.uint8)
        self.lib.orc_unpack(_p(planes), bits, rows, cols, _p(out))
        return out

    def bmma(self, a, a_plane, bt, b_plane, k):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        bt = np.ascontiguousarray(bt, dtype=np.uint64)
        out = np.zeros((a.shape[1], bt.shape[1]), np.int32)
        self.lib.orc_bmma(_p(a), a.shape[0], a.shape[1], a_plane, _p(bt), bt.shape[0], bt.shape[1],
                          b_plane, k, _p(out))
        return out

    def gemm_planes(self, a, bt, k):
        """exact int64 sum_{s,t} 2^(s+t) popc-GEMM (gemm.hpp:94-146, 213-231)"""
        a = np.ascontiguousarray(a, dtype=np.uint64)
        bt = np.ascontiguousarray(bt, dtype=np.uint64)
        out = np.zeros((a.shape[1], bt.shape[1]), np.int64)
        self.lib.orc_gemm_planes(_p(a), a.shape[0], a.shape[1], _p(bt), bt.shape[0], bt.shape[1], k,
                                 _p(out))
        return out

    def gemm_codes(self, a_codes, p, b_codes, q):
        k = a_codes.shape[1]
        return self.gemm_planes(self.bitpack(a_codes, p), self.bitpack(b_codes, q), k)

    def code_rowsums(self, codes):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        out = np.zeros(codes.shape[0], np.int64)
        self.lib.orc_code_rowsums(_p(codes), codes.shape[0], codes.shape[1], _p(out))
        return out

    def zero_point_correct(self, acc, rowsum_a, colsum_b, z_a, z_b, k):
        acc = np.ascontiguousarray(acc, dtype=np.int64)
        m, n = acc.shape
        out = np.zeros((m, n), np.int64)
        self.lib.orc_zero_point_correct(
            _p(acc), m, n, _p(np.ascontiguousarray(rowsum_a, np.int64)),
            _p(np.ascontiguousarray(colsum_b, np.int64)), _p(np.ascontiguousarray(z_a, np.int32)),
            _p(np.ascontiguousarray(z_b, np.int32)), k, _p(out))
        return out

    def quantized_linear(self, act, p, s_a, z_a, wt, q, s_b, z_b, a_per_tensor=False,
                         b_per_tensor=False):
        act = np.ascontiguousarray(act, np.uint8)
        wt = np.ascontiguousarray(wt, np.uint8)
        m, k = act.shape
        n = wt.shape[0]
        out = np.zeros((m, n), np.float64)
        st = self.lib.orc_quantized_linear(
            _p(act), m, p, _p(np.ascontiguousarray(s_a, np.float64)),
            _p(np.ascontiguousarray(z_a, np.int32)), int(a_per_tensor), _p(wt), n, q,
            _p(np.ascontiguousarray(s_b, np.float64)), _p(np.ascontiguousarray(z_b, np.int32)),
            int(b_per_tensor), k, _p(out))
        if st:
            raise ValueError(f"oracle quantized_linear status {st}")
        return out

    def padding_redundancy(self, m, p, mma_m):
        return self.lib.orc_padding_redundancy(m, p, mma_m)

    def fits_int32(self, p, q, k):
        return bool(self.lib.orc_fits_int32(p, q, k))

    def tile_valid(self, BM, BN, BK, WM, WN, WK, p, q):
        return bool(self.lib.orc_tile_valid(BM, BN, BK, WM, WN, WK, p, q))

    def levels(self, bits, scheme):
        return self.lib.orc_levels(bits, scheme)

    def planes(self, bits, scheme):
        return self.lib.orc_planes(bits, scheme)

    def gemm_stats(self, m, n, BM, BN, p, q):
        a = np.zeros(1, np.uint64)
        b = np.zeros(1, np.uint64)
        self.lib.orc_gemm_stats(m, n, BM, BN, p, q, _p(a), _p(b))
        return int(a[0]), int(b[0])

    def dequantize(self, codes, granularity, scales, zps):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.zeros(codes.shape, np.float64)
        self.lib.orc_dequantize(_p(codes), codes.shape[0], codes.shape[1], granularity,
                                _p(np.ascontiguousarray(scales, np.float64)),
                                _p(np.ascontiguousarray(zps, np.int32)), _p(out))
        return out


class RefOracle:
    """oracle/_ref/libabqref.so -- the reference headers themselves."""

    def __init__(self, path: str = REF_LIB_PATH):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_bitpack.argtypes = [_P, _S, _S, _U, _P]
        L.ref_gemm_arbitrary.argtypes = [_P, _U, _S, _P, _U, _S, _S, _P, _U]
        L.ref_gemm_arbitrary_wide.argtypes = [_P, _U, _S, _P, _U, _S, _S, _P]
        L.ref_quantize.argtypes = [_P, _S, _S, _U, _I, _I, C.c_double, C.c_double, _P, _P, _P, _P, _P]
        L.ref_quantized_linear.argtypes = [_P, _S, _U, _I, _I, _P, _P, _P, _S, _U, _I, _I, _P, _P, _S,
                                           _P, _P]
        L.ref_planes_new.restype = C.c_void_p
        L.ref_planes_new.argtypes = [_P, _U, _S, _S]
        L.ref_planes_free.argtypes = [_P]
        L.ref_gemm_arbitrary_h.argtypes = [_P, _P, _P, _U]
        L.ref_gemm_naive_h.argtypes = [_P, _P, _P]
        L.ref_padding_redundancy.restype = C.c_double
        L.ref_padding_redundancy.argtypes = [_S, _U, _S]
        L.ref_fits_int32.argtypes = [_U, _U, _S]
        L.ref_linear_new.restype = C.c_void_p
        L.ref_linear_new.argtypes = [_P, _S, _S, _U, _P, _P, _U]
        L.ref_linear_run.argtypes = [_P, _P, _S, _U, _P]
        L.ref_linear_free.argtypes = [_P]

    def linear(self, wt_codes, w_bits, s_b, z_b, threads=1):
        """Reference linear step with pre-packed weights (ref_shim.cpp
        ref_linear_*); returns run(x_double[m,k], a_bits) -> y[m,n]."""
        wt_codes = np.ascontiguousarray(wt_codes, np.uint8)
        n, k = wt_codes.shape
        s_b = np.ascontiguousarray(s_b, np.float64)
        z_b = np.ascontiguousarray(z_b, np.int32)
        h = self.lib.ref_linear_new(_p(wt_codes), n, k, w_bits, _p(s_b), _p(z_b), threads)
        lib = self.lib

        class _Run:
            def __call__(self_, x, a_bits, out=None):
                x = np.ascontiguousarray(x, np.float64)
                m = x.shape[0]
                if out is None:
                    out = np.zeros((m, n), np.float64)
                st = lib.ref_linear_run(h, _p(x), m, a_bits, _p(out))
                if st:
                    raise ValueError(f"reference linear status {st}")
                return out

            def __del__(self_):
                lib.ref_linear_free(h)

        return _Run()

    @staticmethod
    def available(path: str = REF_LIB_PATH) -> bool:
        return os.path.exists(path)

    def bitpack(self, codes, bits):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        rows, cols = codes.shape
        out = np.zeros((bits, rows, wpr(cols)), np.uint64)
        st = self.lib.ref_bitpack(_p(codes), rows, cols, bits, _p(out))
        if st:
            raise ValueError(f"reference bitpack status {st}")
        return out

    def gemm_arbitrary(self, a, bt, k, threads=0):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        bt = np.ascontiguousarray(bt, dtype=np.uint64)
        out = np.zeros((a.shape[1], bt.shape[1]), np.int32)
        st = self.lib.ref_gemm_arbitrary(_p(a), a.shape[0], a.shape[1], _p(bt), bt.shape[0],
                                         bt.shape[1], k, _p(out), threads)
        if st:
            raise OverflowError(f"reference gemm_arbitrary status {st}")
        return out

    def gemm_arbitrary_wide(self, a, bt, k):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        bt = np.ascontiguousarray(bt, dtype=np.uint64)
        out = np.zeros((a.shape[1], bt.shape[1]), np.int64)
        self.lib.ref_gemm_arbitrary_wide(_p(a), a.shape[0], a.shape[1], _p(bt), bt.shape[0],
                                         bt.shape[1], k, _p(out))
        return out

    def quantize(self, x, bits, scheme=0, granularity=0, alpha=1.0, beta=1.0, comp=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows, cols = x.shape
        groups = 1 if granularity == 0 else rows
        codes = np.zeros((rows, cols), np.uint8)
        scales = np.zeros(groups, np.float64)
        zps = np.zeros(groups, np.int32)
        ca = cb = None
        if comp is not None:
            ca = np.ascontiguousarray(comp[0], dtype=np.float64)
            cb = np.ascontiguousarray(comp[1], dtype=np.float64)
        st = self.lib.ref_quantize(_p(x), rows, cols, bits, scheme, granularity, alpha, beta, _p(ca),
                                   _p(cb), _p(codes), _p(scales), _p(zps))
        if st:
            raise ValueError(f"reference quantize status {st}")
        return codes, scales, zps

    def quantized_linear(self, act, a_bits, a_scheme, a_gran, s_a, z_a, wt, w_bits, w_scheme,
                         w_gran, s_b, z_b):
        act = np.ascontiguousarray(act, np.uint8)
        wt = np.ascontiguousarray(wt, np.uint8)
        m, k = act.shape
        n = wt.shape[0]
        out = np.zeros((m, n), np.float64)
        stats = np.zeros(2, np.uint64)
        st = self.lib.ref_quantized_linear(
            _p(act), m, a_bits, a_scheme, a_gran, _p(np.ascontiguousarray(s_a, np.float64)),
            _p(np.ascontiguousarray(z_a, np.int32)), _p(wt), n, w_bits, w_scheme, w_gran,
            _p(np.ascontiguousarray(s_b, np.float64)), _p(np.ascontiguousarray(z_b, np.int32)), k,
            _p(out), _p(stats))
        if st:
            raise ValueError(f"reference quantized_linear status {st}")
        return out, stats


def load_golden(path: str) -> dict:
    """tests/golden/*.npz -> dict name -> ndarray"""
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


# ---------------------------------------------------------------------------
# large-shape restatement of quantized_linear (gemm.hpp:266-307) for the
# LLaMA-sized parity tests, where the bit-serial C loop would take minutes.
# The code product sum_k a_ik * w_jk is a sum of integers < 2^53 (K * 255^2 at
# K = 2^17 is 2^33), so an fp64 BLAS matmul of the codes is exact; the
# zero-point correction is int64 (gemm.hpp:245-251) and the dequant is
# (s_a[i] * s_b[j]) * corrected in IEEE double, the reference's order
# (gemm.hpp:298).  Pinned against COracle.quantized_linear (tests/test_oracle.py).
# ---------------------------------------------------------------------------
def exact_code_product(a_codes, w_codes) -> np.ndarray:
    a = np.ascontiguousarray(a_codes, np.uint8)
    w = np.ascontiguousarray(w_codes, np.uint8)
    k = a.shape[1]
    assert w.shape[1] == k
    assert k * 255 * 255 < (1 << 53)
    return (a.astype(np.float64) @ w.astype(np.float64).T).astype(np.int64)


def exact_linear(a_codes, s_a, z_a, w_codes, s_b, z_b, acc=None) -> np.ndarray:
    """quantized_linear on codes with per-token (act) / per-channel (weight)
    parameters; float64 [M][N], bit-identical to the reference."""
    a = np.ascontiguousarray(a_codes, np.uint8)
    w = np.ascontiguousarray(w_codes, np.uint8)
    k = a.shape[1]
    if acc is None:
        acc = exact_code_product(a, w)
    ra = a.sum(axis=1, dtype=np.int64)
    cb = w.sum(axis=1, dtype=np.int64)
    za = np.asarray(z_a, np.int64).reshape(-1, 1)
    zb = np.asarray(z_b, np.int64).reshape(1, -1)
    corr = acc - za * cb.reshape(1, -1) - zb * ra.reshape(-1, 1) + k * za * zb
    if np.all(np.abs(corr) < (1 << 31)):
        corr = corr.astype(np.int32)  # the int32 path casts (gemm.hpp:252); values agree either way
    sab = np.asarray(s_a, np.float64).reshape(-1, 1) * np.asarray(s_b, np.float64).reshape(1, -1)
    return sab * corr.astype(np.float64)
