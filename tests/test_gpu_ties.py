"""Rounding ties of the activation ReQuant (quantizer.hpp:205-209: round half
away from zero of the FP64 quotient).  The fp32 fast paths of every ReQuant
site -- the decode GEMV's fused prologue (quant_codes8_f16_band), the
per-token ReQuant kernel feeding the prefill GEMM and the producer-fused
ReQuant (quant_codes8_f16) -- resolve elements inside their tie band with an
FMA test (quant_code_tie) and only fall back to the FP64 division where that
cannot decide.  Activations are built so that many elements are EXACT ties
(step 1: x = n + 1/2) or sit inside the band (step 2/255: the fp16 values whose
quotient is nearest a half-integer); outputs must equal the oracle bit for bit."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _tie_rows(bits, k, rng):
    top = (1 << bits) - 1
    rows = []
    # step 1 (lo = 0, hi = top): exact ties n + 1/2, both signs of distance
    r = np.concatenate([[0.0, float(top)], np.arange(top) + 0.5])
    rows.append(np.resize(rng.permutation(r), k))
    rows[-1][:2] = [0.0, float(top)]
    # step 2 / top (lo = -1, hi = 1): the fp16 values nearest a half-integer quotient
    f = np.concatenate([np.arange(0, 0x3C01, dtype=np.uint16).view(np.float16),
                        -np.arange(1, 0x3C01, dtype=np.uint16).view(np.float16)]).astype(np.float64)
    q = f / (2.0 / top)
    d = np.abs(np.abs(q - np.floor(q)) - 0.5)
    near = f[np.argsort(d)[: max(8, k // 4)]]
    row = rng.choice(near, k)
    row[:2] = [-1.0, 1.0]
    rows.append(row)
    # a negative range with ties: lo = -top, hi = 0 (step 1, zero point top)
    rows.append(-rows[0])
    return np.stack(rows).astype(np.float16)


@pytest.mark.parametrize("bits", [8, 4, 6])
def test_requant_ties_every_site(abq, orc, bits):
    rng = np.random.default_rng(bits)
    k, n = 4096, 1024
    x3 = _tie_rows(bits, k, rng)
    wc = rng.integers(0, 4, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 4, n).astype(np.int32)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 2), sb, zb)
    spec = abq.QuantSpec(bits=bits, granularity=abq.api.PER_TOKEN)
    for m in (1, 3, 16):  # fused decode prologue; ReQuant kernel + prefill GEMM
        x = np.resize(x3, (m, k)) if m <= 3 else np.concatenate([x3] * 6)[:m]
        lin = abq.Linear(w, spec, max_m=m)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), bits, 0, 2)
        want = orc.quantized_linear(ac, bits, sa, za, wc, 2, sb, zb)
        assert np.array_equal(y, want), (bits, m)
    # producer-fused ReQuant: silu(16) * (x / 16) = x exactly in fp16
    m = 3
    gate = torch.full((m, k), 16.0, dtype=torch.float16, device="cuda")
    up = torch.from_numpy((x3.astype(np.float32) / 16).astype(np.float16)).cuda()
    qa = abq.QAct(m, k, spec)
    yprod = torch.empty((m, k), dtype=torch.float16, device="cuda")
    abq.silu_mul_quant(gate, up, spec, out=qa, y_out=yprod)
    assert np.array_equal(yprod.cpu().numpy(), x3)
    lin = abq.Linear(w, spec, max_m=m)
    y = lin(qa, out_dtype=torch.float64).cpu().numpy()
    ac, sa, za = orc.quantize(x3.astype(np.float64), bits, 0, 2)
    assert np.array_equal(y, orc.quantized_linear(ac, bits, sa, za, wc, 2, sb, zb)), bits
