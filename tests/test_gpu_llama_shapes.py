"""GPU parity at the north_star's LLaMA shapes (BASELINE.json configs 3-5,
SURVEY.md 8 config shorthand), through the serving entry point (abq.Linear:
fp16 activations -> ReQuant -> plane GEMV/GEMM -> fused epilogue) against the
oracle: activation codes from the C oracle's quantize (quantizer.hpp:146-213)
and the product from oracle.exact_linear (gemm.hpp:266-307, exact integer
product, reference FP64 dequant order; pinned in tests/test_oracle.py).

  cfg3  W2A4 / W3A8 / W4A8 / W6A6 on every LLaMA-7B linear (fused qkv, o,
        gate/up, down) at M = 1 and M = 128
  cfg4  LLaMA-13B W2A8 decode, the per-GPU shards at G = 2 / 4 / 8
  cfg5  LLaMA-70B W4A4 prefill M = 2048, the per-GPU shards at G = 8,
        including down_proj K = 28672 (the 32-bit corrected-sum regime of the
        tcgen05 epilogue, gemm_tc.cu)
plus the engine's own column sharding (PackedWeights.shard + one Linear per
shard) against the unsharded Linear, bit for bit."""
import numpy as np
import pytest
import torch

from oracle.oracle import exact_linear

pytestmark = pytest.mark.gpu

FP16_RTOL = 2.0 ** -10
FP16_ATOL = 6.1e-5

LLAMA7B = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (11008, 4096), "down": (4096, 11008)}


def _layer(rng, n, k, wbits):
    wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
    return wc, sb, zb


def _check_linear(abq, orc, rng, m, n, k, wbits, abits, tag):
    wc, sb, zb = _layer(rng, n, k, wbits)
    x = rng.standard_normal((m, k)).astype(np.float16)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN), max_m=m)
    xt = torch.from_numpy(x).cuda()
    y64 = lin(xt, out_dtype=torch.float64, check=True).cpu().numpy()
    y16 = lin(xt, out_dtype=torch.float16).cpu().numpy()
    ac, sa, za = orc.quantize(x.astype(np.float64), abits, 0, 2)
    want = exact_linear(ac, sa, za, wc, sb, zb)
    assert np.array_equal(y64, want), tag
    assert np.array_equal(y16, want.astype(np.float16)), tag
    fin = np.abs(want) <= 65504
    err = np.abs(y16.astype(np.float64) - want)
    assert np.all(err[fin] <= FP16_RTOL * np.abs(want[fin]) + FP16_ATOL), tag


@pytest.mark.parametrize("m", [1, 128])
@pytest.mark.parametrize("wbits,abits", [(2, 4), (3, 8), (4, 8), (6, 6)])
def test_cfg3_mixed_precision_llama7b(abq, orc, m, wbits, abits):
    rng = np.random.default_rng(1000 * wbits + 10 * abits + m)
    for name, (n, k) in LLAMA7B.items():
        _check_linear(abq, orc, rng, m, n, k, wbits, abits, (name, m, wbits, abits))


@pytest.mark.parametrize("g", [2, 4, 8])
def test_cfg4_llama13b_w2a8_decode_shards(abq, orc, g):
    rng = np.random.default_rng(4000 + g)
    # q/k/v/o N = K = 5120; gate/up N = 13824 K = 5120; down N = 5120 K = 13824
    for n_full, k in ((5120, 5120), (13824, 5120), (5120, 13824)):
        _check_linear(abq, orc, rng, 1, n_full // g, k, 2, 8, ("13b", n_full, k, g))


@pytest.mark.parametrize("n,k", [(1024, 8192), (128, 8192), (3584, 8192), (1024, 28672)])
def test_cfg5_llama70b_w4a4_prefill_shards(abq, orc, n, k):
    """per-GPU shard of q/o (N=8192/8), k/v (1024/8), gate/up (28672/8) and
    down (8192/8, K=28672) at M=2048 tokens"""
    rng = np.random.default_rng(5000 + n + k)
    _check_linear(abq, orc, rng, 2048, n, k, 4, 4, ("70b", n, k))


@pytest.mark.parametrize("m,n,k,wbits,abits,groups", [
    (1, 13824, 5120, 2, 8, (2, 4, 8)),     # cfg4 gate/up
    (1, 5120, 13824, 2, 8, (2, 8)),        # cfg4 down
    (2048, 8192, 8192, 4, 4, (8,)),        # cfg5 q/o
    (128, 11008, 4096, 4, 4, (2, 4, 8)),   # cfg2 up at M=128
])
def test_engine_shards_concatenate_to_unsharded(abq, m, n, k, wbits, abits, groups):
    """PackedWeights.shard (q contiguous row ranges of the ABQP planes, the
    per-channel slices, re-prepacked per shard) + one Linear per shard: the
    column concatenation equals the unsharded Linear bit for bit (no
    reduction over K)."""
    rng = np.random.default_rng(m + n + k)
    wc, sb, zb = _layer(rng, n, k, wbits)
    x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
    spec = abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
    full = abq.Linear(w, spec, max_m=m)(x, out_dtype=torch.float64)
    for g in groups:
        parts = []
        for r in range(g):
            shard = w.shard(r, g)
            assert shard.planes.rows == n * (r + 1) // g - n * r // g
            parts.append(abq.Linear(shard, spec, max_m=m)(x, out_dtype=torch.float64))
            del shard
        assert torch.equal(torch.cat(parts, dim=1), full), g


def test_resident_layouts_one_per_regime(abq, orc):
    """PackedWeights.resident: one engine layout per serving regime in HBM (the
    planes dropped): decode-only serves m <= 8 and refuses more, prefill-only
    serves any m on the tcgen05 GEMM; outputs equal the full object's."""
    rng = np.random.default_rng(77)
    n, k = 1024, 4096
    wc, sb, zb = _layer(rng, n, k, 4)
    full = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
    spec = abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN)
    dec, pre = full.resident("decode"), full.resident("prefill")
    assert dec.resident_bytes() * 3 == full.resident_bytes() and pre.resident_bytes() * 3 == full.resident_bytes()
    for m in (1, 8, 16, 128):
        x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
        want = abq.Linear(full, spec, max_m=m)(x, out_dtype=torch.float64)
        assert torch.equal(abq.Linear(pre, spec, max_m=m)(x, out_dtype=torch.float64), want), m
        if m <= 8:
            assert torch.equal(abq.Linear(dec, spec, max_m=m)(x, out_dtype=torch.float64), want), m
        else:
            with pytest.raises(abq.ValueError):
                abq.Linear(dec, spec, max_m=m)(x, out_dtype=torch.float64)
