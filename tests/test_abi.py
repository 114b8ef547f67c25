"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/abq_cuda.h declares, its host-only helpers agree with the
oracle, and compute entry points fail loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2408_08554_b200 as abq
from paper_2408_08554_b200 import _lib as L


def test_library_exports_every_header_symbol():
    names = L.header_functions()
    assert len(names) >= 25
    lib = L.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes signature table covers the whole header
    assert sorted(L._SIGNATURES) == names


def test_cpp_headers_cover_c_abi():
    hdr = open(os.path.join(os.path.dirname(L.HEADER_PATH), "abq", "abq.hpp")).read()
    for fn in ["bitpack", "unpack", "bmma", "gemm_arbitrary", "gemm_arbitrary_wide", "gemm_naive",
               "zero_point_correct", "code_rowsums", "quantized_linear", "quantize",
               "fits_int32", "default_tile", "engine_threads", "padding_redundancy"]:
        assert fn + "(" in hdr, fn


def test_host_helpers_match_oracle(orc):
    for p in range(1, 9):
        for q in range(1, 9):
            for k in (1, 63, 64, 4096, 11008, (1 << 15) - 1, 1 << 15, 28672):
                assert abq.fits_int32(p, q, k) == orc.fits_int32(p, q, k)
            t = abq.default_tile(p, q)
            assert (t.BM, t.BN, t.BK, t.WM, t.WN, t.WK) == (64, 64, 512, 32 * p, 32 * q, 128)
            assert t.valid(p, q)
    rng = np.random.default_rng(3)
    for _ in range(300):
        BM, BN = (int(v) for v in rng.integers(1, 130, 2))
        BK = int(rng.choice([100, 128, 256, 384, 512, 640]))
        WM, WN = (int(8 * v + rng.integers(0, 2) * 4) for v in rng.integers(1, 9, 2))
        WK = int(rng.choice([64, 128]))
        p, q = (int(v) for v in rng.integers(1, 9, 2))
        t = abq.TileConfig(BM, BN, BK, WM, WN, WK)
        assert t.valid(p, q) == orc.tile_valid(BM, BN, BK, WM, WN, WK, p, q)
    assert abq.padding_redundancy(1, 1, 8) == 0.875
    assert abq.padding_redundancy(1, 8, 8) == 0.0
    with pytest.raises(abq.ValueError):
        abq.padding_redundancy(0, 1, 8)
    for bits in range(1, 8):
        s = L.QuantSpecC(bits, L.ABQ_BALANCED, 0, 1.0, 1.0)
        assert L.lib().abq_spec_planes(C.byref(s)) == bits + 1 == orc.planes(bits, 2)


def test_invalid_tile_message():
    with pytest.raises(abq.ValueError, match="TileConfig invalid"):
        abq.TileConfig(8, 8, 100, 8, 8, 128).require_valid(1, 1)


def test_compute_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = L.lib()
    st = lib.abq_bitpack(None, 1, 1, 2, None, None)
    assert st == L.ABQ_ERR_CUDA
    assert b"no CUDA device" in lib.abq_last_error()
    with pytest.raises(abq.api.CudaError):
        abq.bitpack(np.zeros((1, 1), np.uint8), 2)
