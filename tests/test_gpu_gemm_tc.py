"""Prefill GEMM on tcgen05 (M >= 9 tokens): plane recombination into u8 codes
in shared memory + UMMA kind::i8 into TMEM.  Bit-exact against the oracle on
ragged shapes (N not a multiple of the 128-channel tile, K multiple of 16 but
not of the 128-wide stage, M not a multiple of the token tile), every weight
plane count, through the fused linear and the raw gemm_arbitrary API."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_tc_linear_ragged(abq, orc):
    rng = np.random.default_rng(21)
    for trial in range(30):
        m = int(rng.integers(9, 300))
        n = int(rng.integers(1, 700))
        k = 16 * int(rng.integers(1, 100))
        wbits, abits = (int(v) for v in rng.integers(1, 9, 2))
        x = (rng.standard_normal((m, k)) * rng.uniform(0.2, 4)).astype(np.float16)
        wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
        sb = rng.uniform(1e-3, 1e-2, n)
        zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
        lin = abq.Linear(w, abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN), max_m=m)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), abits, 0, 2)
        want = orc.quantized_linear(ac, abits, sa, za, wc, wbits, sb, zb)
        assert np.array_equal(y, want), (trial, m, n, k, wbits, abits)


@pytest.mark.parametrize("m,n,k,p,q", [(16, 11008, 4096, 4, 4), (128, 11008, 4096, 4, 4),
                                       (128, 4096, 4096, 8, 2), (128, 11008, 4096, 8, 8),
                                       (200, 1024, 11008, 6, 6), (2048, 512, 1024, 4, 4)])
def test_tc_gemm_llama_shapes(abq, orc, m, n, k, p, q):
    rng = np.random.default_rng(m * 7 + n)
    a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
    b = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
    got = abq.gemm_arbitrary(abq.bitpack(a, p), abq.bitpack(b, q), abq.default_tile(p, q)).cpu().numpy()
    want = a.astype(np.int64) @ b.astype(np.int64).T  # exact integer product
    assert np.array_equal(got, want)


def test_tc_gemm_random_raw(abq, orc):
    rng = np.random.default_rng(22)
    for trial in range(40):
        m = int(rng.integers(16, 260))
        n = int(rng.integers(1, 400))
        k = 16 * int(rng.integers(1, 60))
        p, q = (int(v) for v in rng.integers(1, 9, 2))
        a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
        b = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
        got = abq.gemm_arbitrary(abq.bitpack(a, p), abq.bitpack(b, q), abq.default_tile(p, q)).cpu().numpy()
        assert np.array_equal(got, orc.gemm_codes(a, p, b, q)), (trial, m, n, k, p, q)


def test_tc_variant_matches_popc(abq):
    """same call under the forced AND+popcount variant gives the same bits"""
    rng = np.random.default_rng(23)
    a = rng.integers(0, 16, (64, 1024), dtype=np.uint8)
    b = rng.integers(0, 16, (300, 1024), dtype=np.uint8)
    pa, pb = abq.bitpack(a, 4), abq.bitpack(b, 4)
    tc = abq.gemm_arbitrary(pa, pb, abq.default_tile(4, 4))
    abq.api.set_gemv_variant("popc")
    try:
        popc = abq.gemm_arbitrary(pa, pb, abq.default_tile(4, 4))
    finally:
        abq.api.set_gemv_variant("auto")
    assert torch.equal(tc, popc)


@pytest.mark.parametrize("m,n,k,p,q", [(128, 1000, 4096, 4, 4), (37, 300, 1000, 8, 8), (128, 512, 2048, 8, 2),
                                       (9, 77, 300, 2, 2)])
def test_btc_gemm_matches_oracle(abq, orc, m, n, k, p, q):
    """b1 tensor-core comparator (mma.sync m16n8k256 .b1 and.popc) is exact"""
    rng = np.random.default_rng(m + n + k)
    a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
    b = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
    got = abq.gemm_btc(abq.bitpack(a, p), abq.bitpack(b, q)).cpu().numpy()
    assert np.array_equal(got, orc.gemm_codes(a, p, b, q))


@pytest.mark.parametrize("m,n,k,wbits,abits", [
    (128, 11008, 4096, 4, 4),   # LLaMA-7B up: 86 row-tiles -> 148 CTAs, <= 2 contributors per tile
    (9, 128, 32, 3, 5),         # one row-tile, two k-blocks -> 2 CTAs
    (200, 300, 48 * 16, 2, 8),  # 3 row-tiles, 6 k-blocks, token tile 256
    (64, 5000, 3 * 128, 8, 8),  # odd k-block count
    (33, 19000, 1024, 5, 3),    # row-tiles (149) >= SMs: no stream-K
    (100, 640, 11008, 6, 6),    # long K, 5 row-tiles -> 10 CTAs of ~43 k-blocks
])
def test_tc_stream_k(abq, orc, m, n, k, wbits, abits):
    """stream-K prefill GEMM (one token tile, row-tiles < SMs): bit-exact against
    the oracle, repeated calls (the hand-off flags reset themselves), a
    smaller m through the same workspace, and equal to the one-CTA-per-tile
    schedule (abq_set_gemm_schedule(CLASSIC))."""
    abq.api.set_gemm_schedule("stream_k")
    rng = np.random.default_rng(m + n + k)
    wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN), max_m=m)
    for mm in (m, max(9, m // 2 + 1), m):
        x = (rng.standard_normal((mm, k)) * 2).astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        ac, sa, za = orc.quantize(x.astype(np.float64), abits, 0, 2)
        want = orc.quantized_linear(ac, abits, sa, za, wc, wbits, sb, zb)
        for rep in range(2):
            y = lin(xd, out_dtype=torch.float64).cpu().numpy()
            assert np.array_equal(y, want), (mm, rep)
        y16 = lin(xd, out_dtype=torch.float16).cpu().numpy()
        assert np.array_equal(y16, want.astype(np.float16)), mm
    abq.api.set_gemm_schedule("classic")
    try:
        assert np.array_equal(lin(xd, out_dtype=torch.float64).cpu().numpy(), want)
    finally:
        abq.api.set_gemm_schedule("auto")


def test_linear_workspace_serves_every_m_up_to_max_m(abq, orc):
    """A Linear sized for max_m accepts every m <= max_m: the workspace need is
    monotone in m (the stream-K partial tiles are sized for min(m, 256))."""
    lib = abq._lib.lib()
    n, k = 11008, 4096
    needs = [lib.abq_linear_workspace_bytes(m, n, k, 4) for m in range(1, 2049, 7)] + \
        [lib.abq_linear_workspace_bytes(2048, n, k, 4)]
    assert all(a <= b for a, b in zip(needs, needs[1:]))
    rng = np.random.default_rng(31)
    wc = rng.integers(0, 16, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 16, n).astype(np.int32)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN), max_m=2048)
    for m in (1, 128, 200, 2048):
        x = rng.standard_normal((m, k)).astype(np.float16)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), 4, 0, 2)
        assert np.array_equal(y, orc.quantized_linear(ac, 4, sa, za, wc, 4, sb, zb)), m
