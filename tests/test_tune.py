"""Tune API (tune.hpp:17-192) on the GPU build: candidate enumeration pinned to
the reference's own output (tests/golden/tune, written by the unmodified
enumerate_tile_candidates / padding_redundancy / tops_of through
oracle/gen_tune_golden.cpp), the reference's error behaviour, and -- on the
GPU -- autotune over tile candidates (bit-for-bit verified) and over the
engine's own schedules for a resident layer (autotune_linear)."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2408_08554_b200 as abq

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "tune", "candidates.json")


def _digest(cands):
    return hashlib.sha256("".join("%d,%d,%d,%d,%d,%d;" % (t.BM, t.BN, t.BK, t.WM, t.WN, t.WK)
                                  for t in cands).encode()).hexdigest()


def test_candidates_match_reference():
    cases = json.load(open(GOLDEN))
    n = 0
    for c in cases:
        if "tops_of" in c:
            m, nn, k, us, want = c["tops_of"]
            assert abq.tops_of(m, nn, k, us) == want
            continue
        got = abq.enumerate_tile_candidates(c["p"], c["q"], c["m"], 4096, 4096)
        assert len(got) == c["count"], c
        assert [got[0].BM, got[0].BN, got[0].BK, got[0].WM, got[0].WN, got[0].WK] == c["first"]
        assert [got[-1].BM, got[-1].BN, got[-1].BK, got[-1].WM, got[-1].WN, got[-1].WK] == c["last"]
        assert _digest(got) == c["sha256"], c
        assert abq.padding_redundancy(c["m"], c["p"], abq.TileConfig.mma_m) == c["padding"]
        n += 1
    assert n == 150


def test_candidates_properties():
    """test_tune.cpp:25-48: every candidate valid, no duplicates, GEMV (M=1)
    candidates carry the minimal row padding"""
    for p, q in [(1, 1), (3, 5), (8, 8)]:
        c = abq.enumerate_tile_candidates(p, q, 1, 4096, 4096)
        assert all(t.valid(p, q) for t in c)
        keys = [(t.BM, t.BN, t.BK, t.WM, t.WN) for t in c]
        assert len(keys) == len(set(keys))
        pads = {abq.api._total_row_padding(1, p, t.BM, 8) for t in c}
        assert len(pads) == 1


def test_tune_errors():
    with pytest.raises(abq.ValueError, match="p,q must be in"):
        abq.enumerate_tile_candidates(0, 4, 1, 64, 64)
    with pytest.raises(abq.ValueError, match="p,q must be in"):
        abq.enumerate_tile_candidates(4, 9, 1, 64, 64)
    with pytest.raises(abq.ValueError, match="no candidates"):
        abq.autotune([], None, None)
    with pytest.raises(abq.ValueError, match="at least 3 trials"):
        abq.autotune([abq.default_tile(1, 1)], None, None, trials=2)
    assert abq.BenchRecord.csv_header() == "config_id,BM,BN,BK,WM,WN,p,q,M,N,K,median_us,tops"
    r = abq.BenchRecord("x", 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 1.5, 2.5)
    assert r.csv_row() == "x,1,2,3,4,5,6,7,8,9,10,1.5,2.5"


def test_gemm_schedule_setting():
    assert abq.get_gemm_schedule() == "auto"
    for s in ("classic", "stream_k", "auto"):
        abq.set_gemm_schedule(s)
        assert abq.get_gemm_schedule() == s
    with pytest.raises(abq.ValueError):
        abq.set_gemm_schedule("split")


@pytest.mark.gpu
def test_autotune_tiles(orc):
    rng = np.random.default_rng(5)
    m, n, k, p, q = 40, 70, 300, 3, 5
    a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
    b = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
    cands = abq.enumerate_tile_candidates(p, q, m, n, k)[:5]
    res = abq.autotune(cands, abq.bitpack(a, p), abq.bitpack(b, q), trials=3)
    assert res.best in cands and len(res.records) == len(cands)
    assert all(r.median_us > 0 and r.tops > 0 and (r.M, r.N, r.K, r.p, r.q) == (m, n, k, p, q)
               for r in res.records)
    got = abq.gemm_arbitrary(abq.bitpack(a, p), abq.bitpack(b, q), res.best).cpu().numpy()
    assert np.array_equal(got, orc.gemm_codes(a, p, b, q))


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [(1, 4096, 4096), (128, 2048, 1024), (64, 300, 512)])
def test_autotune_linear(abq, orc, m, n, k):
    import torch
    rng = np.random.default_rng(m + n)
    wbits, abits = 4, 4
    wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN), max_m=m)
    x = (rng.standard_normal((m, k)) * 2).astype(np.float16)
    xd = torch.from_numpy(x).cuda()
    try:
        res = abq.autotune_linear(lin, xd, trials=3, out_dtype=torch.float64)
        names = [r.config_id for r in res.records]
        assert res.best in names and (names[0] == "auto" if m <= 8 else names[0] == "classic")
        ac, sa, za = orc.quantize(x.astype(np.float64), abits, 0, 2)
        want = orc.quantized_linear(ac, abits, sa, za, wc, wbits, sb, zb)
        assert np.array_equal(lin(xd, out_dtype=torch.float64).cpu().numpy(), want)  # winner selected
    finally:
        abq.set_gemv_variant("auto")
        abq.set_gemm_schedule("auto")


def test_tile_maps_to_distinct_engine_schedules():
    """TileConfig -> engine schedule (abq_tile_engine_plan):
    BM caps the token tile, BK == 128 selects stream-K; the reference's own
    candidate lists therefore time different kernels."""
    from paper_2408_08554_b200.api import tile_engine_plan
    assert tile_engine_plan(abq.TileConfig(64, 64, 512, 64, 64, 128)) == (64, "classic")
    assert tile_engine_plan(abq.TileConfig(16, 64, 128, 32, 64, 128)) == (16, "stream_k")
    assert tile_engine_plan(abq.TileConfig(1, 8, 256, 8, 8, 128))[0] == 1
    plans = {tile_engine_plan(t) for t in abq.api.enumerate_tile_candidates(4, 4, 128, 11008, 4096)}
    assert len(plans) >= 2, plans
