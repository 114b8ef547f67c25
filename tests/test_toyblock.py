"""Model-level drop-in: the reference toy block's forward_fp and
forward_quant (toyblock.hpp:191-282) against golden outputs of the UNMODIFIED
reference (tests/golden/toy/toy.json, oracle/gen_toy_golden.cpp) on the same
seeded weights and input.  The real-arithmetic parts run in the reference's
operation order and every projection goes through the GPU engine (quantize +
quantized_linear, FP64-exact), so the block output is expected bit for bit;
the reference's own model-level pins use 1e-9, the bound
asserted here besides the exact-match count."""
import json
import os

import numpy as np
import pytest

from paper_2408_08554_b200 import model

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "toy", "toy.json")))


def _mat(name):
    m = G[name]
    return np.array(m["data"], dtype=np.float64).reshape(m["rows"], m["cols"])


def _block():
    return model.ToyBlock(*(_mat(n) for n in ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown")), heads=G["heads"])


def test_forward_fp_matches_reference():
    b = _block()
    assert (b.dim, b.hidden) == (G["dim"], G["hidden"])
    out, trace = model.forward_fp(b, _mat("x"))
    assert np.array_equal(out, _mat("forward_fp"))
    assert model.first_token_attention_share(trace) == G["share_fp"]


def test_toyblock_errors():
    b = _block()
    with pytest.raises(model.api.ShapeError, match="input width"):
        model.forward_fp(b, np.zeros((2, 3)))
    with pytest.raises(model.api.ValueError, match="no attention maps"):
        model.first_token_attention_share(model.ForwardTrace())


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["quant_w4a4", "quant_w8a8", "quant_w3a6_params"])
def test_forward_quant_matches_reference(cfg):
    b = _block()
    if cfg == "quant_w3a6_params":
        specs = model.BlockSpecs.make(3, 6)
        p = b.init_params()
        for n in model.LAYERS:
            p.layers[n] = model.LayerParams(np.array(G["s_" + n]), 0.9, 0.95)
        p.comp_a, p.comp_b, p.gamma = np.array(G["comp_a"]), np.array(G["comp_b"]), 1
    else:
        bits = int(cfg[-1])
        specs, p = model.BlockSpecs.make(bits, bits), b.init_params()
    out, trace = model.forward_quant(b, _mat("x"), specs, p)
    want = _mat(cfg)
    assert np.max(np.abs(out - want)) <= 1e-9
    assert np.array_equal(out, want), f"{np.count_nonzero(out != want)} of {out.size} differ (within 1e-9)"
    assert [e.layer for e in trace.events] == list(model.LAYERS)
    assert abs(model.first_token_attention_share(trace) - G["share_" + cfg]) <= 1e-12
