"""Pin the C restatement (oracle/abq_oracle.c) against the reference's own
golden vectors (tests/golden/reference_cases.npz, produced by the reference
headers via oracle/_ref) and, where oracle/_ref exists, against the reference
on fresh random inputs.  CPU only."""
import hashlib

import numpy as np
import pytest

from conftest import family, seeded_codes


# ---- bit planes (test_bitkernel.cpp:36-66) ---------------------------------
def test_bitpack_golden(golden, orc):
    for bits in range(1, 9):
        c = golden[f"bitpack/{bits}/codes"]
        planes = orc.bitpack(c, bits)
        assert np.array_equal(planes, golden[f"bitpack/{bits}/planes"])
        assert np.array_equal(orc.unpack(planes, c.shape[1]), c)
        # tail bits past cols are zero (bitplane.hpp:13-14)
        tail = c.shape[1] % 64
        if tail:
            assert not np.any(planes[:, :, -1] >> np.uint64(tail))


def test_bitpack_rejects_out_of_range(orc):
    bad = np.zeros((2, 3), np.uint8)
    bad[1, 2] = 4
    with pytest.raises(ValueError, match="index 5"):
        orc.bitpack(bad, 2)


def test_bmma_golden(golden, orc):
    a, b = golden["bmma/a"], golden["bmma/b"]
    pa, pb = orc.bitpack(a, 3), orc.bitpack(b, 2)
    for s in range(3):
        for t in range(2):
            assert np.array_equal(orc.bmma(pa, s, pb, t, a.shape[1]), golden[f"bmma/out/{s}_{t}"])


# ---- engine (test_bitkernel.cpp:68-180, acceptance.cpp:29-104) -------------
@pytest.mark.parametrize("fam", ["gemm23", "accept42"])
def test_gemm_golden_families(golden, orc, fam):
    ids = family(golden, fam)
    assert len(ids) >= 60
    for i in ids:
        p, q = (int(v) for v in golden[f"{fam}/{i}/pq"])
        a, b = golden[f"{fam}/{i}/a"], golden[f"{fam}/{i}/b"]
        got = orc.gemm_codes(a, p, b, q)
        assert np.array_equal(got, golden[f"{fam}/{i}/out"].astype(np.int64)), (fam, i)
        # and the plain int64 code matmul (the reference tests' oracle)
        assert np.array_equal(got, a.astype(np.int64) @ b.astype(np.int64).T)


def test_naive_tile_overflow_golden(golden, orc):
    a, b = golden["naive24/a"], golden["naive24/b"]
    got = orc.gemm_codes(a, 5, b, 3)
    assert np.array_equal(got, golden["naive24/naive"])
    assert np.array_equal(got, golden["naive24/tiled"])
    a, b = golden["tile26/a"], golden["tile26/b"]
    assert np.array_equal(orc.gemm_codes(a, 3, b, 5), golden["tile26/out"])
    a, b = golden["tile43/a"], golden["tile43/b"]
    assert np.array_equal(orc.gemm_codes(a, 5, b, 3), golden["tile43/out"])
    # overflow boundary K = 2^15 at p=q=8 (test_bitkernel.cpp:90-102)
    assert orc.fits_int32(8, 8, (1 << 15) - 1) and not orc.fits_int32(8, 8, 1 << 15)
    assert int(golden["overflow25/threw"][0]) == 1
    a, b = golden["overflow25/a"], golden["overflow25/b"]
    assert np.array_equal(orc.gemm_codes(a, 8, b, 8), golden["overflow25/wide"])


def test_zero_point_golden(golden, orc):
    for i in family(golden, "zp27"):
        g = lambda n: golden[f"zp27/{i}/{n}"]  # noqa: E731
        a, b = g("a"), g("b")
        acc = orc.gemm_codes(a, 4, b, 4)
        assert np.array_equal(acc, g("acc"))
        corr = orc.zero_point_correct(acc, orc.code_rowsums(a), orc.code_rowsums(b), g("za"), g("zb"),
                                      a.shape[1])
        assert np.array_equal(corr, g("corrected"))
        signed = (a.astype(np.int64) - g("za")[:, None]) @ (b.astype(np.int64) - g("zb")[:, None]).T
        assert np.array_equal(corr, signed)


def test_quantized_linear_golden(golden, orc):
    qa = lambda n: golden[f"qlinear28/qa/{n}"]  # noqa: E731
    qw = lambda n: golden[f"qlinear28/qw/{n}"]  # noqa: E731
    codes_a, sa, za = orc.quantize(golden["qlinear28/x"], 5, 0, 2)
    codes_w, sw, zw = orc.quantize(golden["qlinear28/w"], 3, 0, 1)
    assert np.array_equal(codes_a, qa("codes")) and np.array_equal(sa, qa("scales"))
    assert np.array_equal(za, qa("zero_points"))
    assert np.array_equal(codes_w, qw("codes")) and np.array_equal(sw, qw("scales"))
    assert np.array_equal(zw, qw("zero_points"))
    y = orc.quantized_linear(codes_a, 5, sa, za, codes_w, 3, sw, zw)
    assert np.array_equal(y, golden["qlinear28/out"])  # bit-identical doubles
    # test_bitkernel.cpp:165: equals the dequantized product within 1e-9
    deq = orc.dequantize(codes_a, 2, sa, za) @ orc.dequantize(codes_w, 1, sw, zw).T
    assert np.max(np.abs(y - deq)) < 1e-9
    assert tuple(golden["qlinear28/stats"]) == orc.gemm_stats(6, 9, 64, 64, 5, 3)


def test_stats_law(golden, orc):
    # test_bitkernel.cpp:170-180 with TileConfig{32,32,128,32,32,128}
    assert tuple(golden["stats29/stats"]) == orc.gemm_stats(70, 70, 32, 32, 2, 3) == (9, 54)
    assert np.array_equal(orc.gemm_codes(golden["stats29/a"], 2, golden["stats29/b"], 3),
                          golden["stats29/out"])


# ---- quantizer (test_quantizer.cpp) -----------------------------------------
def test_quantizer_alpha_beta_comp_golden(golden, orc):
    for i in family(golden, "quant7"):
        g = lambda n: golden[f"quant7/{i}/{n}"]  # noqa: E731
        bits, scheme, gran = (int(v) for v in g("meta"))
        alpha, beta = g("alpha_beta")
        codes, scales, zps = orc.quantize(g("x"), bits, scheme, gran, alpha, beta,
                                          (g("comp_a"), g("comp_b")))
        assert np.array_equal(codes, g("q/codes")), i
        assert np.array_equal(scales, g("q/scales")), i
        assert np.array_equal(zps, g("q/zero_points")), i


def test_quantizer_roundtrip_balanced_golden(golden, orc):
    for i in family(golden, "quant11"):
        g = lambda n: golden[f"quant11/{i}/{n}"]  # noqa: E731
        bits, scheme, gran = (int(v) for v in g("meta"))
        codes, scales, zps = orc.quantize(g("x"), bits, scheme, gran)
        assert np.array_equal(codes, g("q/codes")) and np.array_equal(scales, g("q/scales"))
        assert np.array_equal(zps, g("q/zero_points"))
        back = orc.dequantize(codes, gran, scales, zps)
        assert np.all(np.abs(back - g("x")) <= scales[:, None] / 2 + 1e-12)
    codes, scales, zps = orc.quantize(golden["balanced3/x"], 2, 2, 0)
    assert np.array_equal(codes, golden["balanced3/q/codes"])
    assert set(np.unique(codes.astype(int) - zps[0])) == {-2, -1, 0, 1, 2}
    assert orc.planes(2, 2) == 3 and orc.levels(2, 2) == 5
    codes, scales, zps = orc.quantize(golden["degenerate/x"], 4, 0, 0)
    assert scales[0] == 1.0 and zps[0] == 0 and np.all(codes == 3)


# ---- scalar API (tune.hpp, gemm.hpp) ----------------------------------------
def test_padding_and_tiles(orc):
    assert orc.padding_redundancy(1, 1, 8) == 0.875
    assert orc.padding_redundancy(1, 8, 8) == 0.0
    for m in range(1, 17):
        for p in range(1, 9):
            e = p * m
            pad = -(-e // 8) * 8
            assert orc.padding_redundancy(m, p, 8) == (pad - e) / pad
    assert not orc.tile_valid(8, 8, 100, 8, 8, 128, 1, 1)
    assert not orc.tile_valid(8, 8, 128, 8, 8, 64, 1, 1)
    assert not orc.tile_valid(8, 8, 128, 12, 8, 128, 1, 1)
    assert not orc.tile_valid(512, 512, 128, 8, 8, 128, 1, 1)
    assert orc.tile_valid(64, 64, 512, 32, 32, 128, 1, 1)


# ---- large numpy-seeded cases vs stored reference outputs ------------------
def test_big_cases_golden(golden, orc):
    a, w = seeded_codes(1001, 1, 4096, 8), seeded_codes(1002, 4096, 4096, 2)
    assert np.array_equal(orc.gemm_codes(a, 8, w, 2), golden["big/cfg1_w2a8/out"])
    a, w = seeded_codes(1003, 1, 4096, 4), seeded_codes(1004, 11008, 4096, 4)
    assert np.array_equal(orc.gemm_codes(a, 4, w, 4), golden["big/cfg2_w4a4_m1/out"])


def test_big_quantized_linear_golden(golden, orc):
    x = np.random.default_rng(1007).standard_normal((1, 4096)).astype(np.float16).astype(np.float64)
    wf = np.random.default_rng(1008).standard_normal((4096, 4096)) * 0.02
    ac, asc, az = orc.quantize(x, 8, 0, 2)
    wc, wsc, wz = orc.quantize(wf, 2, 0, 1)
    assert np.array_equal(ac, golden["big/qlinear_cfg1/act_codes"])
    assert hashlib.sha256(wc.tobytes()).digest() == golden["big/qlinear_cfg1/wt_sha256"].tobytes()
    assert np.array_equal(wsc, golden["big/qlinear_cfg1/wt_scales"])
    y = orc.quantized_linear(ac, 8, asc, az, wc, 2, wsc, wz)
    assert np.array_equal(y, golden["big/qlinear_cfg1/out"])


# ---- oracle vs the reference itself on fresh random inputs ------------------
def test_oracle_matches_reference_random(orc, ref):
    rng = np.random.default_rng(7)
    for _ in range(40):
        m, n, k = (int(v) for v in rng.integers(1, 90, size=3))
        k = int(rng.integers(1, 700))
        p, q = (int(v) for v in rng.integers(1, 9, size=2))
        a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
        b = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
        pa, pb = orc.bitpack(a, p), orc.bitpack(b, q)
        assert np.array_equal(pa, ref.bitpack(a, p))
        assert np.array_equal(orc.gemm_planes(pa, pb, k), ref.gemm_arbitrary(pa, pb, k))
    for _ in range(40):
        rows, cols = (int(v) for v in rng.integers(1, 40, size=2))
        x = rng.standard_normal((rows, cols)) * rng.uniform(0.1, 5)
        scheme = int(rng.integers(0, 3))
        bits = int(rng.integers(1, 8 if scheme == 2 else 9))
        gran = int(rng.integers(0, 3))
        alpha, beta = rng.uniform(0.5, 1.0, size=2)
        comp = (rng.standard_normal(rows), rng.standard_normal(cols)) if rng.random() < 0.5 else None
        got = orc.quantize(x, bits, scheme, gran, alpha, beta, comp)
        want = ref.quantize(x, bits, scheme, gran, alpha, beta, comp)
        for g_, w_ in zip(got, want):
            assert np.array_equal(g_, w_)
    # quantized_linear at a shape that needs the wide path (p+q+log2(K+1) > 31)
    a = rng.integers(0, 256, (2, 40000), dtype=np.uint8)
    b = rng.integers(0, 256, (3, 40000), dtype=np.uint8)
    sa, za = rng.uniform(0.01, 0.1, 2), rng.integers(0, 256, 2).astype(np.int32)
    sb, zb = rng.uniform(0.01, 0.1, 3), rng.integers(0, 256, 3).astype(np.int32)
    y_ref, _ = ref.quantized_linear(a, 8, 0, 2, sa, za, b, 8, 0, 1, sb, zb)
    assert np.array_equal(orc.quantized_linear(a, 8, sa, za, b, 8, sb, zb), y_ref)


# ---- the large-shape numpy restatement used by the LLaMA-shape GPU tests ----
def test_exact_linear_matches_oracle_and_golden(golden, orc):
    from oracle.oracle import exact_code_product, exact_linear
    rng = np.random.default_rng(17)
    for _ in range(30):
        m, n = (int(v) for v in rng.integers(1, 40, size=2))
        k = int(rng.integers(1, 900))
        p, q = (int(v) for v in rng.integers(1, 9, size=2))
        x = rng.standard_normal((m, k)) * rng.uniform(0.1, 5)
        ac, sa, za = orc.quantize(x, p, 0, 2)
        wc = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
        sb = rng.uniform(1e-3, 1e-2, n)
        zb = rng.integers(0, 1 << q, n).astype(np.int32)
        assert np.array_equal(exact_code_product(ac, wc), orc.gemm_codes(ac, p, wc, q).astype(np.int64))
        assert np.array_equal(exact_linear(ac, sa, za, wc, sb, zb), orc.quantized_linear(ac, p, sa, za, wc, q, sb, zb))
    # the wide regime (p + q + log2(K+1) > 31) too
    a = rng.integers(0, 256, (2, 40000), dtype=np.uint8)
    b = rng.integers(0, 256, (3, 40000), dtype=np.uint8)
    sa, za = rng.uniform(0.01, 0.1, 2), rng.integers(0, 256, 2).astype(np.int32)
    sb, zb = rng.uniform(0.01, 0.1, 3), rng.integers(0, 256, 3).astype(np.int32)
    assert np.array_equal(exact_linear(a, sa, za, b, sb, zb), orc.quantized_linear(a, 8, sa, za, b, 8, sb, zb))
    # and the reference-emitted LLaMA-shaped golden outputs
    a, w = seeded_codes(1001, 1, 4096, 8), seeded_codes(1002, 4096, 4096, 2)
    assert np.array_equal(exact_code_product(a, w), golden["big/cfg1_w2a8/out"])
    a, w = seeded_codes(1003, 1, 4096, 4), seeded_codes(1004, 11008, 4096, 4)
    assert np.array_equal(exact_code_product(a, w), golden["big/cfg2_w4a4_m1/out"])
