"""On-disk weight formats: ABQT / ABQP / ABQZ files written by
the reference's own abq::io writers (tests/golden/io, made by
tests/golden/make_io_golden.py) parse, re-serialise byte-identically, agree
with each other (ABQP = bitpack of the ABQT codes), and fail like io.hpp on
bad input.  The GPU test loads the bundle into HBM and runs the engine."""
import io
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _bytes(name):
    with open(os.path.join(GOLD, name), "rb") as f:
        return f.read()


@pytest.fixture(scope="module")
def abqio():
    from paper_2408_08554_b200 import io as abqio
    return abqio


def test_abqt_roundtrip_and_fields(abqio):
    for name, (rows, cols, bits, gran) in {"wt_pc4.abqt": (5, 70, 4, 1), "wt_pt3.abqt": (3, 129, 3, 0)}.items():
        raw = _bytes(name)
        q = abqio.read_quantized(io.BytesIO(raw))
        assert q.codes.shape == (rows, cols) and q.spec.bits == bits and q.spec.granularity == gran
        assert q.scales.size == (1 if gran == 0 else rows) and np.all(q.scales > 0)
        assert int(q.codes.max()) < (1 << bits)
        out = io.BytesIO()
        abqio.write_quantized(out, q)
        assert out.getvalue() == raw, name


def test_abqp_is_bitpack_of_abqt_codes(abqio):
    q = abqio.read_quantized(io.BytesIO(_bytes("wt_pc4.abqt")))
    raw = _bytes("wt_pc4.abqp")
    p = abqio.read_planes(io.BytesIO(raw))
    assert (p.planes, p.rows, p.cols) == (q.spec.planes(), 5, 70)
    assert np.array_equal(p.words, abqio.host_bitpack(q.codes, q.spec.planes()).words)
    out = io.BytesIO()
    abqio.write_planes(out, p)
    assert out.getvalue() == raw


def test_abqz_bundle(abqio):
    raw = _bytes("bundle.abqz")
    layers = abqio.read_bundle(io.BytesIO(raw))
    assert [n for n, _, _ in layers] == ["up", "down"]
    for _, q, p in layers:
        assert np.array_equal(p.words, abqio.host_bitpack(q.codes, q.spec.planes()).words)
    out = io.BytesIO()
    abqio.write_bundle(out, layers)
    assert out.getvalue() == raw


def test_io_errors_like_reference(abqio):
    from paper_2408_08554_b200 import IoError, ValueError
    raw = bytearray(_bytes("wt_pc4.abqt"))
    with pytest.raises(IoError, match="bad magic, expected ABQT"):
        abqio.read_quantized(io.BytesIO(b"ABQP" + bytes(raw[4:])))
    bad_ver = bytearray(raw)
    bad_ver[4] = 9
    with pytest.raises(IoError, match="ABQT: unsupported version"):
        abqio.read_quantized(io.BytesIO(bytes(bad_ver)))
    with pytest.raises(IoError, match="ABQT: truncated code block"):
        abqio.read_quantized(io.BytesIO(bytes(raw[:-3])))
    with pytest.raises(IoError, match="unexpected end of file"):
        abqio.read_quantized(io.BytesIO(bytes(raw[:12])))
    hi = bytearray(raw)
    hi[-1] = 200  # > 15: code out of range for 4 bits
    with pytest.raises(ValueError, match="code out of range at flat index 349"):
        abqio.read_quantized(io.BytesIO(bytes(hi)))
    praw = bytearray(_bytes("wt_pc4.abqp"))
    praw[15] = 7  # words_per_row field
    with pytest.raises(IoError, match="ABQP: inconsistent words_per_row"):
        abqio.read_planes(io.BytesIO(bytes(praw)))


@pytest.mark.gpu
def test_bundle_to_engine(abq, orc, abqio):
    import torch
    layers = abqio.read_bundle(os.path.join(GOLD, "bundle.abqz"))
    weights = abqio.load_bundle(os.path.join(GOLD, "bundle.abqz"))
    rng = np.random.default_rng(3)
    for name, q, _ in layers:
        w = weights[name]
        m = 3
        x = rng.standard_normal((m, q.cols())).astype(np.float16)
        lin = abq.Linear(w, abq.QuantSpec(bits=6, granularity=abq.api.PER_TOKEN), max_m=m)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), 6, 0, 2)
        sb = np.broadcast_to(q.scales, (q.rows(),)) if q.scales.size == 1 else q.scales
        zb = np.broadcast_to(q.zero_points, (q.rows(),)) if q.zero_points.size == 1 else q.zero_points
        want = orc.quantized_linear(ac, 6, sa, za, q.codes, q.spec.bits, np.ascontiguousarray(sb),
                                    np.ascontiguousarray(zb, dtype=np.int32))
        assert np.array_equal(y, want), name
