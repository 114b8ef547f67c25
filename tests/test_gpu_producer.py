"""Producer-fused ReQuant: RMSNorm / SiLU(gate)*up with the
per-token ReQuant of their fp16 output fused in (producer.cu), consumed by the
decode GEMV (abq_linear_qact).

Pins:
* the producer's fp16 output y against a torch fp32 reference of the same op
  (LLaMA RMSNorm / SiLU*up), within fp16 rounding;
* the codes, s_a, z_a and code row sums against the C oracle's quantize
  (quantizer.hpp:146-213) applied to that y -- bit-exact;
* the consumer's output against oracle.exact_linear on those codes
  (gemm.hpp:266-307) -- bit-exact, FP64 and fp16;
* one producer feeding several projections (q/k/v), back to back;
* validation: per-tensor spec, m > 8, non-finite outputs."""
import numpy as np
import pytest
import torch

from oracle.oracle import exact_linear

pytestmark = pytest.mark.gpu


def _weights(abq, rng, n, k, wbits):
    wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
    return wc, sb, zb, abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)


def _check_qact(abq, orc, qa, y, abits):
    """codes / stats of qa == oracle quantize(y) (per token, asymmetric)"""
    ac, sa, za = orc.quantize(y.astype(np.float64), abits, 0, 2)
    assert np.array_equal(qa.codes_matrix(), ac)
    assert np.array_equal(qa.scales.cpu().numpy(), sa)
    assert np.array_equal(qa.zero_points.cpu().numpy(), za)
    assert np.array_equal(qa.rowsums.cpu().numpy(), ac.astype(np.int64).sum(1))
    return ac, sa, za


@pytest.mark.parametrize("m,k,abits", [(1, 4096, 4), (1, 4096, 8), (2, 5120, 8), (5, 4096, 4), (8, 1024, 6),
                                       (1, 11008, 8), (3, 13824, 4)])
def test_rmsnorm_quant_matches_torch_and_oracle(abq, orc, m, k, abits):
    rng = np.random.default_rng(m * 1000 + k + abits)
    x = torch.from_numpy((rng.standard_normal((m, k)) * 2).astype(np.float16)).cuda()
    gain = torch.from_numpy(rng.uniform(0.5, 1.5, k).astype(np.float16)).cuda()
    eps = 1e-5
    spec = abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN)
    y = torch.empty_like(x)
    qa = abq.rmsnorm_quant(x, gain, eps, spec, y_out=y, check=True)
    xf = x.float()
    want = gain * (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).half()
    torch.testing.assert_close(y, want, rtol=2 ** -9, atol=1e-3)
    _check_qact(abq, orc, qa, y.cpu().numpy(), abits)


@pytest.mark.parametrize("m,k,abits", [(1, 11008, 8), (1, 11008, 4), (4, 13824, 8), (8, 2048, 3)])
def test_silu_mul_quant_matches_torch_and_oracle(abq, orc, m, k, abits):
    rng = np.random.default_rng(7 * m + k + abits)
    gate = torch.from_numpy((rng.standard_normal((m, k)) * 3).astype(np.float16)).cuda()
    up = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
    spec = abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN)
    y = torch.empty_like(gate)
    qa = abq.silu_mul_quant(gate, up, spec, y_out=y, check=True)
    want = torch.nn.functional.silu(gate.float()).half() * up
    torch.testing.assert_close(y, want, rtol=2 ** -9, atol=1e-3)
    _check_qact(abq, orc, qa, y.cpu().numpy(), abits)


@pytest.mark.parametrize("m,wbits,abits", [(1, 4, 4), (1, 2, 8), (2, 8, 8), (8, 4, 4), (3, 3, 5)])
def test_producer_feeds_several_projections(abq, orc, m, wbits, abits):
    """one RMSNorm+ReQuant -> q, k, v decode GEMVs (LLaMA-7B shapes, N=4096
    each), back to back without synchronisation; each equals the oracle."""
    rng = np.random.default_rng(100 * m + wbits)
    k = 4096
    x = torch.from_numpy(rng.standard_normal((m, k)).astype(np.float16)).cuda()
    gain = torch.from_numpy(rng.uniform(0.8, 1.2, k).astype(np.float16)).cuda()
    spec = abq.QuantSpec(bits=abits, granularity=abq.api.PER_TOKEN)
    projs = [_weights(abq, rng, 4096, k, wbits) for _ in range(3)]
    lins = [abq.Linear(w, spec, max_m=m) for *_, w in projs]
    y = torch.empty_like(x)
    for rep in range(2):
        n0 = abq.launch_count()
        qa = abq.rmsnorm_quant(x, gain, 1e-6, spec, y_out=y)
        outs = [lin(qa, out_dtype=torch.float64) for lin in lins]
        outs16 = [lin(qa, out_dtype=torch.float16) for lin in lins]
        assert abq.launch_count() - n0 == 1 + 6  # one producer, one GEMV launch per projection
        qa.raise_if_nonfinite()
        ac, sa, za = _check_qact(abq, orc, qa, y.cpu().numpy(), abits)
        for (wc, sb, zb, _), o, o16 in zip(projs, outs, outs16):
            want = exact_linear(ac, sa, za, wc, sb, zb)
            assert np.array_equal(o.cpu().numpy(), want), rep
            assert np.array_equal(o16.cpu().numpy(), want.astype(np.float16)), rep


def test_silu_producer_feeds_down_proj(abq, orc):
    """gate / up GEMVs -> SiLU*up+ReQuant -> down GEMV (LLaMA-7B MLP, W4A4, M=1)"""
    rng = np.random.default_rng(3)
    spec = abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN)
    wc, sb, zb, w = _weights(abq, rng, 4096, 11008, 4)
    down = abq.Linear(w, spec, max_m=1)
    gate = torch.from_numpy(rng.standard_normal((1, 11008)).astype(np.float16)).cuda()
    up = torch.from_numpy(rng.standard_normal((1, 11008)).astype(np.float16)).cuda()
    y = torch.empty_like(gate)
    qa = abq.silu_mul_quant(gate, up, spec, y_out=y)
    out = down(qa, out_dtype=torch.float64).cpu().numpy()
    ac, sa, za = _check_qact(abq, orc, qa, y.cpu().numpy(), 4)
    assert np.array_equal(out, exact_linear(ac, sa, za, wc, sb, zb))


def test_producer_validation_and_nonfinite(abq):
    k = 1024
    x = torch.zeros((2, k), dtype=torch.float16, device="cuda")
    gain = torch.ones(k, dtype=torch.float16, device="cuda")
    with pytest.raises(abq.ValueError):
        abq.QAct(2, k, abq.QuantSpec(bits=4, granularity=abq.api.PER_TENSOR))
    spec = abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN)
    with pytest.raises(abq.ValueError):
        abq.rmsnorm_quant(torch.zeros((9, k), dtype=torch.float16, device="cuda"), gain, 1e-6, spec)
    up = torch.ones((2, k), dtype=torch.float16, device="cuda")
    gate = torch.zeros((2, k), dtype=torch.float16, device="cuda")
    gate[1, 37] = float("inf")
    with pytest.raises(abq.ValueError, match=r"\(1,37\)"):
        abq.silu_mul_quant(gate, up, spec, check=True)
    qa = abq.silu_mul_quant(gate, up, spec)  # launch-only: recorded, raised on request
    with pytest.raises(abq.ValueError, match=r"\(1,37\)"):
        qa.raise_if_nonfinite()
    abq.rmsnorm_quant(x, gain, 1e-6, spec, check=True)  # all-zero rows: degenerate range, fine
    with pytest.raises(abq.ShapeError):
        rng = np.random.default_rng(0)
        *_, w = _weights(abq, rng, 64, 512, 4)
        abq.Linear(w, spec, max_m=2)(abq.rmsnorm_quant(x, gain, 1e-6, spec))


def test_concat_weights_equal_separate_projections(abq, orc):
    """PackedWeights.concat (fused q/k/v, gate/up): the concatenated launch's
    column blocks equal the separate projections, decode and prefill."""
    rng = np.random.default_rng(5)
    spec = abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN)
    parts = [_weights(abq, rng, n, 1024, 4) for n in (512, 128, 384)]
    cat = abq.PackedWeights.concat([w for *_, w in parts])
    for m in (1, 3, 40):
        x = torch.from_numpy(rng.standard_normal((m, 1024)).astype(np.float16)).cuda()
        y = abq.Linear(cat, spec, max_m=m)(x, out_dtype=torch.float64)
        sep = torch.cat([abq.Linear(w, spec, max_m=m)(x, out_dtype=torch.float64) for *_, w in parts], dim=1)
        assert torch.equal(y, sep), m
