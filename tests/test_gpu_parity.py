"""GPU parity: the sm_100a engine (through the C-ABI) against the reference's
golden vectors and the pinned oracle.  Integer / byte / index results must be
bit-exact; the FP64 API-parity output must be bit-identical; the fp16
performance output must equal round-to-nearest-fp16 of the reference double,
and in any case stay within the stated tolerance
    |y_gpu - y_ref| <= 2^-10 * |y_ref| + 6.1e-5.
Mirrors test_bitkernel.cpp / test_quantizer.cpp / acceptance.cpp."""
import numpy as np
import pytest
import torch

from conftest import family, seeded_codes

pytestmark = pytest.mark.gpu

FP16_RTOL = 2.0 ** -10
FP16_ATOL = 6.1e-5


def planes_np(abq, m):
    return m.numpy()


def cpu(t):
    return t.cpu().numpy()


# ---- bit planes (test_bitkernel.cpp:36-66) ---------------------------------
def test_bitpack_roundtrip_and_error(abq, golden):
    for bits in range(1, 9):
        c = golden[f"bitpack/{bits}/codes"]
        m = abq.bitpack(c, bits)
        assert m.planes == bits
        assert np.array_equal(m.numpy(), golden[f"bitpack/{bits}/planes"])
        assert np.array_equal(cpu(abq.unpack(m)), c)
    bad = np.zeros((2, 3), np.uint8)
    bad[1, 2] = 4
    with pytest.raises(abq.ValueError, match=r"\(1,2\)"):
        abq.bitpack(bad, 2)
    with pytest.raises(abq.ValueError):
        abq.bitpack(bad, 9)


def test_bmma_triple_loop(abq, golden):
    a, b = golden["bmma/a"], golden["bmma/b"]
    pa, pb = abq.bitpack(a, 3), abq.bitpack(b, 2)
    for s in range(3):
        for t in range(2):
            assert np.array_equal(cpu(abq.bmma(pa, s, pb, t)), golden[f"bmma/out/{s}_{t}"])


# ---- engine -----------------------------------------------------------------
@pytest.mark.parametrize("fam", ["gemm23", "accept42"])
def test_gemm_arbitrary_golden(abq, golden, fam):
    for i in family(golden, fam):
        p, q = (int(v) for v in golden[f"{fam}/{i}/pq"])
        a, b = golden[f"{fam}/{i}/a"], golden[f"{fam}/{i}/b"]
        got = abq.gemm_arbitrary(abq.bitpack(a, p), abq.bitpack(b, q), abq.default_tile(p, q))
        assert got.dtype == torch.int32
        assert np.array_equal(cpu(got), golden[f"{fam}/{i}/out"]), (fam, i, p, q, a.shape, b.shape)


def test_naive_agrees_with_tiled(abq, golden):
    pa, pb = abq.bitpack(golden["naive24/a"], 5), abq.bitpack(golden["naive24/b"], 3)
    assert np.array_equal(cpu(abq.gemm_naive(pa, pb)), golden["naive24/naive"])
    assert np.array_equal(cpu(abq.gemm_arbitrary(pa, pb, abq.default_tile(5, 3))), golden["naive24/tiled"])


def test_overflow_guard_and_wide(abq, golden):
    assert abq.fits_int32(8, 8, (1 << 15) - 1) and not abq.fits_int32(8, 8, 1 << 15)
    pa, pb = abq.bitpack(golden["overflow25/a"], 8), abq.bitpack(golden["overflow25/b"], 8)
    with pytest.raises(abq.OverflowError, match="exceeds 31"):
        abq.gemm_arbitrary(pa, pb, abq.default_tile(8, 8))
    wide = abq.gemm_arbitrary_wide(pa, pb, abq.default_tile(8, 8))
    assert cpu(wide)[0, 0] == golden["overflow25/wide"][0, 0]


def test_validation_order(abq):
    a = abq.bitpack(np.zeros((2, 10), np.uint8), 2)
    b = abq.bitpack(np.zeros((2, 11), np.uint8), 2)
    bad_tile = abq.TileConfig(8, 8, 100, 8, 8, 128)
    with pytest.raises(abq.ShapeError, match="shared K dimension differs"):
        abq.gemm_arbitrary(a, b, bad_tile)  # shape before tile
    big = abq.bitpack(np.zeros((1, 1 << 15), np.uint8), 8)
    with pytest.raises(abq.ValueError, match="TileConfig invalid"):
        abq.gemm_arbitrary(big, big, bad_tile)  # tile before overflow


def test_tile_transparency(abq, golden):
    pa, pb = abq.bitpack(golden["tile26/a"], 3), abq.bitpack(golden["tile26/b"], 5)
    want = golden["tile26/out"]
    for bm in (8, 16, 64):
        for bk in (128, 256, 512):
            got = abq.gemm_arbitrary(pa, pb, abq.TileConfig(bm, 32, bk, 24, 40, 128))
            assert np.array_equal(cpu(got), want)
    pa, pb = abq.bitpack(golden["tile43/a"], 5), abq.bitpack(golden["tile43/b"], 3)
    assert np.array_equal(cpu(abq.gemm_arbitrary(pa, pb, abq.default_tile(5, 3))), golden["tile43/out"])


def test_zero_point_correction(abq, golden):
    for i in family(golden, "zp27"):
        g = lambda n: golden[f"zp27/{i}/{n}"]  # noqa: E731
        a, b = g("a"), g("b")
        acc = abq.gemm_arbitrary(abq.bitpack(a, 4), abq.bitpack(b, 4), abq.default_tile(4, 4))
        assert np.array_equal(cpu(acc), g("acc"))
        corr = abq.zero_point_correct(acc, abq.code_rowsums(a), abq.code_rowsums(b), g("za"), g("zb"),
                                      a.shape[1])
        assert np.array_equal(cpu(corr), g("corrected"))
        corr64 = abq.zero_point_correct(acc.long(), abq.code_rowsums(a), abq.code_rowsums(b),
                                        g("za"), g("zb"), a.shape[1])
        assert np.array_equal(cpu(corr64), g("corrected"))


def test_quantized_linear_bit_identical(abq, golden):
    qa = abq.quantize(golden["qlinear28/x"], abq.QuantSpec(bits=5, granularity=abq.api.PER_TOKEN))
    qw = abq.quantize(golden["qlinear28/w"], abq.QuantSpec(bits=3, granularity=abq.api.PER_CHANNEL))
    assert np.array_equal(cpu(qa.codes), golden["qlinear28/qa/codes"])
    assert np.array_equal(cpu(qa.scales), golden["qlinear28/qa/scales"])
    assert np.array_equal(cpu(qw.codes), golden["qlinear28/qw/codes"])
    assert np.array_equal(cpu(qw.zero_points), golden["qlinear28/qw/zero_points"])
    stats = abq.GemmStats()
    y = abq.quantized_linear(qa, qw, stats)
    assert y.dtype == torch.float64
    assert np.array_equal(cpu(y), golden["qlinear28/out"])
    deq = cpu(abq.dequantize(qa)) @ cpu(abq.dequantize(qw)).T
    assert np.max(np.abs(cpu(y) - deq)) < 1e-9
    assert (stats.block_tiles, stats.plane_pair_products) == tuple(golden["qlinear28/stats"])


def test_gemm_stats_law(abq, golden):
    stats = abq.GemmStats()
    out = abq.gemm_arbitrary(abq.bitpack(golden["stats29/a"], 2), abq.bitpack(golden["stats29/b"], 3),
                             abq.TileConfig(32, 32, 128, 32, 32, 128), stats)
    assert (stats.block_tiles, stats.plane_pair_products) == (9, 54)
    assert np.array_equal(cpu(out), golden["stats29/out"])


# ---- quantizer (test_quantizer.cpp) -----------------------------------------
def test_quantize_alpha_beta_compensation(abq, golden):
    for i in family(golden, "quant7"):
        g = lambda n: golden[f"quant7/{i}/{n}"]  # noqa: E731
        bits, scheme, gran = (int(v) for v in g("meta"))
        alpha, beta = (float(v) for v in g("alpha_beta"))
        q = abq.quantize(g("x"), abq.QuantSpec(bits, scheme, gran, alpha, beta), (g("comp_a"), g("comp_b")))
        assert np.array_equal(cpu(q.codes), g("q/codes")), i
        assert np.array_equal(cpu(q.scales), g("q/scales")), i
        assert np.array_equal(cpu(q.zero_points), g("q/zero_points")), i


def test_quantize_roundtrip_balanced_degenerate(abq, golden):
    for i in family(golden, "quant11"):
        g = lambda n: golden[f"quant11/{i}/{n}"]  # noqa: E731
        bits, scheme, gran = (int(v) for v in g("meta"))
        q = abq.quantize(g("x"), abq.QuantSpec(bits, scheme, gran))
        assert np.array_equal(cpu(q.codes), g("q/codes"))
        assert np.array_equal(cpu(q.scales), g("q/scales"))
    q = abq.quantize_balanced(golden["balanced3/x"], 2)
    assert np.array_equal(cpu(q.codes), golden["balanced3/q/codes"])
    assert q.spec.planes() == 3 and q.spec.levels() == 5
    q = abq.quantize(golden["degenerate/x"], abq.QuantSpec(bits=4))
    assert cpu(q.scales)[0] == 1.0 and cpu(q.zero_points)[0] == 0 and np.all(cpu(q.codes) == 3)


def test_quantize_rejects_non_finite_and_bad_spec(abq):
    x = np.ones((2, 2))
    x[1, 1] = np.nan
    with pytest.raises(abq.ValueError, match=r"\(1,1\)"):
        abq.quantize(x, abq.QuantSpec())
    for spec in (abq.QuantSpec(bits=0), abq.QuantSpec(bits=9), abq.QuantSpec(alpha=0.0),
                 abq.QuantSpec(bits=16), abq.QuantSpec(bits=8, scheme=abq.api.BALANCED)):
        with pytest.raises(abq.ValueError):
            abq.quantize(np.ones((1, 1)), spec)


# ---- fp16 activations: fused ReQuant + BitPacking (K1) ----------------------
def test_quant_pack_act_fp16_matches_oracle(abq, orc):
    rng = np.random.default_rng(11)
    for m, k, bits in [(1, 4096, 8), (3, 4096, 4), (8, 11008, 8), (5, 130, 3), (16, 64, 6), (2, 1, 8)]:
        x = (rng.standard_normal((m, k)) * rng.uniform(0.1, 3)).astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        spec = abq.QuantSpec(bits=bits, granularity=abq.api.PER_TOKEN)
        planes = torch.empty((bits, m, (k + 63) // 64), dtype=torch.int64, device="cuda")
        sa = torch.empty(m, dtype=torch.float64, device="cuda")
        za = torch.empty(m, dtype=torch.int32, device="cuda")
        ra = torch.empty(m, dtype=torch.int64, device="cuda")
        codes = torch.empty((m, k), dtype=torch.uint8, device="cuda")
        import ctypes as C
        sc = spec.c()
        st = abq._lib.lib().abq_quant_pack_act(xd.data_ptr(), 0, m, k, C.byref(sc), planes.data_ptr(),
                                               sa.data_ptr(), za.data_ptr(), ra.data_ptr(),
                                               codes.data_ptr(), None,
                                               torch.cuda.current_stream().cuda_stream)
        assert st == 0
        oc, osc, oz = orc.quantize(x.astype(np.float64), bits, 0, 2)
        assert np.array_equal(cpu(codes), oc)
        assert np.array_equal(cpu(sa), osc) and np.array_equal(cpu(za), oz)
        assert np.array_equal(planes.cpu().numpy().view(np.uint64), orc.bitpack(oc, bits))
        assert np.array_equal(cpu(ra), orc.code_rowsums(oc))


# ---- random shapes vs the oracle (acceptance.cpp:29-52 style) ---------------
def test_random_shapes_vs_oracle(abq, orc):
    rng = np.random.default_rng(42)
    for _ in range(150):
        m = int(rng.integers(1, 40))
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, 1200))
        p, q = (int(v) for v in rng.integers(1, 9, 2))
        a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
        b = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
        want = orc.gemm_codes(a, p, b, q)
        got = abq.gemm_arbitrary_wide(abq.bitpack(a, p), abq.bitpack(b, q), abq.default_tile(p, q))
        assert np.array_equal(cpu(got), want), (m, n, k, p, q)
        if abq.fits_int32(p, q, k):
            got32 = abq.gemm_arbitrary(abq.bitpack(a, p), abq.bitpack(b, q), abq.default_tile(p, q))
            assert np.array_equal(cpu(got32), want)


# ---- LLaMA-shaped cases vs stored reference outputs --------------------------
def test_cfg1_w2a8_gemv_bit_exact(abq, golden):
    a, w = seeded_codes(1001, 1, 4096, 8), seeded_codes(1002, 4096, 4096, 2)
    got = abq.gemm_arbitrary(abq.bitpack(a, 8), abq.bitpack(w, 2), abq.default_tile(8, 2))
    assert np.array_equal(cpu(got), golden["big/cfg1_w2a8/out"])


def test_cfg2_w4a4_and_w8a8(abq, golden):
    import hashlib
    a, w = seeded_codes(1003, 1, 4096, 4), seeded_codes(1004, 11008, 4096, 4)
    got = abq.gemm_arbitrary(abq.bitpack(a, 4), abq.bitpack(w, 4), abq.default_tile(4, 4))
    assert np.array_equal(cpu(got), golden["big/cfg2_w4a4_m1/out"])
    a, w = seeded_codes(1005, 4, 4096, 8), seeded_codes(1006, 11008, 4096, 8)
    got = cpu(abq.gemm_arbitrary(abq.bitpack(a, 8), abq.bitpack(w, 8), abq.default_tile(8, 8)))
    assert hashlib.sha256(got.astype(np.int32).tobytes()).digest() == golden["big/cfg2_w8a8_m4/sha256"].tobytes()


def _cfg1_linear_inputs(abq):
    x = np.random.default_rng(1007).standard_normal((1, 4096)).astype(np.float16)
    wf = np.random.default_rng(1008).standard_normal((4096, 4096)) * 0.02
    qw = abq.quantize(wf, abq.QuantSpec(bits=2, granularity=abq.api.PER_CHANNEL))
    return x, qw


def test_end_to_end_linear_cfg1(abq, golden):
    """fp16 x -> ReQuant+BitPack -> W2A8 GEMV -> fused epilogue; F64 output
    bit-identical to the reference quantized_linear, fp16 output equal to its
    round-to-nearest and within the stated tolerance."""
    import hashlib
    x, qw = _cfg1_linear_inputs(abq)
    assert hashlib.sha256(cpu(qw.codes).tobytes()).digest() == golden["big/qlinear_cfg1/wt_sha256"].tobytes()
    w = abq.PackedWeights.from_quantized(qw)
    spec = abq.QuantSpec(bits=8, granularity=abq.api.PER_TOKEN)
    lin = abq.Linear(w, spec, max_m=8)
    xd = torch.from_numpy(x).cuda()
    want = golden["big/qlinear_cfg1/out"]
    y64 = cpu(lin(xd, out_dtype=torch.float64))
    assert np.array_equal(y64, want)
    y16 = cpu(lin(xd, out_dtype=torch.float16)).astype(np.float64)
    assert np.array_equal(y16, want.astype(np.float16).astype(np.float64))
    assert np.all(np.abs(y16 - want) <= FP16_RTOL * np.abs(want) + FP16_ATOL)
    # asynchronous (no host sync) path gives the same result
    y16b = cpu(lin(xd, out_dtype=torch.float16, check=False)).astype(np.float64)
    assert np.array_equal(y16b, y16)


@pytest.mark.parametrize("m", [1, 4, 8, 16, 128])
@pytest.mark.parametrize("wbits,abits", [(4, 4), (8, 8), (2, 8), (2, 4), (3, 8), (4, 8), (6, 6)])
def test_linear_shapes_vs_oracle(abq, orc, m, wbits, abits):
    rng = np.random.default_rng(1000 * m + 10 * wbits + abits)
    n, k = (11008, 4096) if m <= 8 else (1024, 4096)
    x = rng.standard_normal((m, k)).astype(np.float16)
    wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN), max_m=m)
    y = cpu(lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64))
    ac, sa, za = orc.quantize(x.astype(np.float64), abits, 0, 2)
    want = orc.quantized_linear(ac, abits, sa, za, wc, wbits, sb, zb)
    assert np.array_equal(y, want)
