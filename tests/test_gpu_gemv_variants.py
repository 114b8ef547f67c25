"""Both decode-GEMV variants (AND+popcount on CUDA cores, and weight planes on
the int8 tensor pipe) must produce bit-identical results to the oracle on
ragged shapes: N not a multiple of the 16-row tile, K not a multiple of the
256-element block, every (p, q) pair, per-token and per-tensor activations,
fp16 / fp32 / fp64 inputs, the stream-K (workspace) and row-tile paths."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["popc", "recomb"])
def variant(request, abq):
    abq.api.set_gemv_variant(request.param)
    yield request.param
    abq.api.set_gemv_variant("auto")


def _case(rng, m, n, k, wbits, abits, xdtype=np.float16):
    x = (rng.standard_normal((m, k)) * rng.uniform(0.2, 4)).astype(xdtype)
    wc = rng.integers(0, 1 << wbits, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wbits, n).astype(np.int32)
    return x, wc, sb, zb


def test_linear_ragged_shapes(abq, orc, variant):
    rng = np.random.default_rng(5)
    for trial in range(60):
        m = int(rng.integers(1, 9))
        n = int(rng.integers(1, 700))
        k = int(rng.integers(1, 1500))
        wbits, abits = (int(v) for v in rng.integers(1, 9, 2))
        x, wc, sb, zb = _case(rng, m, n, k, wbits, abits)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, wbits), sb, zb)
        gran = abq.api.PER_TENSOR if trial % 5 == 0 else abq.api.PER_TOKEN
        lin = abq.Linear(w, abq.QuantSpec(bits=abits, granularity=gran), max_m=m)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), abits, 0, gran)
        want = orc.quantized_linear(ac, abits, sa, za, wc, wbits, sb, zb, a_per_tensor=gran == 0)
        assert np.array_equal(y, want), (trial, m, n, k, wbits, abits, gran)


def test_linear_planes_ragged(abq, orc, variant):
    """activation planes given (abq_linear_planes): row-tile split, no workspace"""
    rng = np.random.default_rng(6)
    for trial in range(40):
        m = int(rng.integers(1, 9))
        n = int(rng.integers(1, 900))
        k = int(rng.integers(1, 2100))
        p, q = (int(v) for v in rng.integers(1, 9, 2))
        a = rng.integers(0, 1 << p, (m, k), dtype=np.uint8)
        wc = rng.integers(0, 1 << q, (n, k), dtype=np.uint8)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, q), np.ones(n), np.zeros(n, np.int32))
        pa = abq.bitpack(a, p)
        sa = torch.ones(m, dtype=torch.float64, device="cuda")
        za = torch.zeros(m, dtype=torch.int32, device="cuda")
        got = abq.linear_planes(pa, sa, za, abq.code_rowsums(a), w, torch.int64).cpu().numpy()
        assert np.array_equal(got, orc.gemm_codes(a, p, wc, q)), (trial, m, n, k, p, q)


@pytest.mark.parametrize("xdtype", [np.float16, np.float32, np.float64])
def test_linear_input_dtypes(abq, orc, variant, xdtype):
    rng = np.random.default_rng(7)
    x, wc, sb, zb = _case(rng, 3, 333, 1000, 4, 8, xdtype)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=8, granularity=abq.api.PER_TOKEN), max_m=3)
    y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
    ac, sa, za = orc.quantize(x.astype(np.float64), 8, 0, 2)
    assert np.array_equal(y, orc.quantized_linear(ac, 8, sa, za, wc, 4, sb, zb))


def test_linear_symmetric_balanced_schemes(abq, orc, variant):
    rng = np.random.default_rng(8)
    for scheme, bits in [(abq.api.SYMMETRIC, 4), (abq.api.BALANCED, 3), (abq.api.SYMMETRIC, 1)]:
        x, wc, sb, zb = _case(rng, 2, 200, 512, 2, 8)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, 2), sb, zb)
        spec = abq.QuantSpec(bits=bits, scheme=scheme, granularity=abq.api.PER_TOKEN)
        lin = abq.Linear(w, spec, max_m=2)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), bits, scheme, 2)
        want = orc.quantized_linear(ac, spec.planes(), sa, za, wc, 2, sb, zb)
        assert np.array_equal(y, want), (scheme, bits)


def test_nonfinite_activation_reported(abq, variant):
    rng = np.random.default_rng(9)
    x, wc, sb, zb = _case(rng, 2, 64, 256, 4, 4)
    x[1, 17] = np.inf
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN), max_m=2)
    with pytest.raises(abq.ValueError, match=r"\(1,17\)"):
        lin(torch.from_numpy(x).cuda(), check=True)
    # the next clean call succeeds (status word and accumulators are reset)
    x[1, 17] = 0.5
    lin(torch.from_numpy(x).cuda(), check=True)
    # serving default (check=False): launch-only, the report is read later
    x[1, 17] = -np.inf
    lin(torch.from_numpy(x).cuda())
    with pytest.raises(abq.ValueError, match=r"\(1,17\)"):
        lin.raise_if_nonfinite()
    x[1, 17] = 0.25
    lin(torch.from_numpy(x).cuda())
    lin.raise_if_nonfinite()


def test_linear_argument_checks(abq, variant):
    rng = np.random.default_rng(12)
    x, wc, sb, zb = _case(rng, 2, 64, 256, 4, 4)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN), max_m=4)
    xt = torch.from_numpy(x).cuda()
    with pytest.raises(abq.ShapeError, match="inner dimensions"):
        lin(torch.zeros((2, 255), dtype=torch.float16, device="cuda"))
    with pytest.raises(abq.ValueError, match="contiguous"):
        lin(torch.zeros((256, 2), dtype=torch.float16, device="cuda").t())
    with pytest.raises(abq.ShapeError):
        lin(xt, out=torch.empty((2, 63), dtype=torch.float16, device="cuda"))
    with pytest.raises(abq.ShapeError):
        lin(xt, out=torch.empty((64, 2), dtype=torch.float16, device="cuda").t())
    with pytest.raises(abq.ValueError):
        lin(xt.cpu())


def test_repeated_calls_are_deterministic(abq, variant):
    """self-cleaning cross-CTA accumulators: identical results call after call"""
    rng = np.random.default_rng(10)
    x, wc, sb, zb = _case(rng, 1, 11008, 4096, 4, 4)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN), max_m=1)
    xd = torch.from_numpy(x).cuda()
    first = lin(xd, out_dtype=torch.float64).clone()
    for _ in range(20):
        assert torch.equal(lin(xd, out_dtype=torch.float64, check=False), first)


def test_chained_layers_back_to_back(abq, orc):
    """layers of different shapes launched back to back on one stream (the
    PDL chain: each launch starts while its predecessor drains, and waits for
    it before reading activations), outputs read only at the end: every layer
    equals the oracle, repeatedly."""
    rng = np.random.default_rng(11)
    m, k = 2, 1024
    layers = []
    for n, wb, ab in ((700, 4, 4), (300, 2, 8), (513, 8, 3)):
        x, wc, sb, zb = _case(rng, m, n, k, wb, ab)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
        lin = abq.Linear(w, abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m)
        ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
        layers.append((torch.from_numpy(x).cuda(), lin, orc.quantized_linear(ac, ab, sa, za, wc, wb, sb, zb)))
    for rep in range(3):
        outs = [lin(xt, out_dtype=torch.float64) for xt, lin, _ in layers * 2]
        for (xt, lin, want), y in zip(layers * 2, outs):
            assert np.array_equal(y.cpu().numpy(), want), rep


@pytest.mark.parametrize("m,n,k,wb,ab", [
    (1, 4096, 11008, 2, 8),   # LLaMA-7B down_proj, W2A8 decode (fused ReQuant, K not a 4096 multiple)
    (3, 5120, 5120, 4, 4),    # LLaMA-13B q_proj, 3 tokens
    (8, 2048, 4096, 4, 4),    # 8 tokens: ReQuant kernel + GEMV (PDL pair)
    (1, 1024, 13824, 6, 6),   # LLaMA-13B down_proj K, W6A6 (non power-of-two slices)
])
def test_serving_gemv_llama_shapes(abq, orc, m, n, k, wb, ab):
    rng = np.random.default_rng(m * 131 + k)
    x, wc, sb, zb = _case(rng, m, n, k, wb, ab)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
    lin = abq.Linear(w, abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m)
    xt = torch.from_numpy(x).cuda()
    n0 = abq.launch_count()
    y64 = lin(xt, out_dtype=torch.float64).cpu().numpy()
    # the serving decode path: ONE launch with the ReQuant fused into the GEMV
    # prologue (K * tokens small enough), else the ReQuant kernel + the GEMV
    fused = k * (1 if m == 1 else 2 if m == 2 else 4 if m <= 4 else 8) <= 16384
    assert abq.launch_count() - n0 == (1 if fused else 2), (m, k)
    y16 = lin(xt, out_dtype=torch.float16).cpu().numpy()
    ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
    want = orc.quantized_linear(ac, ab, sa, za, wc, wb, sb, zb)
    assert np.array_equal(y64, want)
    assert np.array_equal(y16, want.astype(np.float16))


def test_serving_linear_random_shapes_vs_oracle(abq, orc):
    """Fuzz of the serving entry point (fused-ReQuant decode GEMV with its TMA
    producer warp, ring refills, ragged N / K tails; the tcgen05 prefill GEMM)
    against the oracle, bit for bit: 60 random (m, n, k, q, p) incl. shares
    larger than the ring."""
    rng = np.random.default_rng(2024)
    cases = []
    for i in range(60):
        if i % 10 == 0:    # shares larger than the ring (refills), decode
            m, n, k = int(rng.integers(1, 9)), int(rng.integers(9000, 24000)), int(rng.integers(512, 1024)) * 8
        elif i % 4 == 0:   # prefill
            m, n, k = int(rng.integers(9, 160)), int(rng.integers(1, 1500)), int(rng.integers(1, 512)) * 8
        else:              # decode, ragged N, K multiple of 8 or not (ReQuant-kernel path)
            m, n = int(rng.integers(1, 9)), int(rng.integers(1, 3000))
            k = int(rng.integers(1, 1600)) * 8 if i % 3 else int(rng.integers(1, 9000))
        wb, ab = (int(v) for v in rng.integers(1, 9, 2))
        cases.append((m, n, k, wb, ab))
    from oracle.oracle import exact_linear
    for (m, n, k, wb, ab) in cases:
        x, wc, sb, zb = _case(rng, m, n, k, wb, ab)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
        lin = abq.Linear(w, abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m)
        y = lin(torch.from_numpy(x).cuda(), out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
        want = exact_linear(ac, sa, za, wc, sb, zb)
        assert np.array_equal(y, want), (m, n, k, wb, ab)


@pytest.mark.parametrize("m,n,k,wb,ab", [(1, 11008, 4096, 4, 4), (3, 1000, 4100, 2, 8), (16, 512, 2048, 4, 4)])
def test_host_linear_end_to_end(abq, orc, m, n, k, wb, ab):
    """HostLinear.step(): pinned host activations staged by a kernel over PCIe
    (abq_stage_in, incl. a byte tail), the linear's epilogue writing y into
    pinned host memory; several calls back to back (PDL-chained) each equal
    the oracle."""
    rng = np.random.default_rng(m + n + k)
    hosts, wants = [], []
    for rep in range(3):
        x, wc, sb, zb = _case(rng, m, n, k, wb, ab)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
        h = abq.HostLinear(abq.Linear(w, abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m), m)
        h.x_host.copy_(torch.from_numpy(x))
        ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
        hosts.append(h)
        wants.append(orc.quantized_linear(ac, ab, sa, za, wc, wb, sb, zb).astype(np.float16))
    for h in hosts:
        h.step()
    torch.cuda.synchronize()
    for h, want in zip(hosts, wants):
        assert np.array_equal(h.y_host.numpy(), want)


@pytest.mark.parametrize("m,n,k,wb,ab", [(1, 11008, 4096, 4, 4), (16, 512, 2048, 4, 4)])
def test_graphed_host_linear_end_to_end(abq, orc, m, n, k, wb, ab):
    """GraphedHostLinear.step(): HostLinear's step replayed from a CUDA graph;
    new host activations written between replays are picked up (the graph
    reads the pinned buffer), each result equals the oracle."""
    rng = np.random.default_rng(7 * m + n)
    x, wc, sb, zb = _case(rng, m, n, k, wb, ab)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
    g = abq.GraphedHostLinear(abq.Linear(w, abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m), m)
    for rep in range(3):
        x = (rng.standard_normal((m, k)) * (rep + 1)).astype(np.float16)
        g.x_host.copy_(torch.from_numpy(x))
        g.step()
        torch.cuda.synchronize()
        ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
        want = orc.quantized_linear(ac, ab, sa, za, wc, wb, sb, zb).astype(np.float16)
        assert np.array_equal(g.y_host.numpy(), want), rep


def test_prefetch_next_hint_is_transparent(abq, orc):
    """abq_weights.next (Linear.prefetch_next): a cycle of decode layers of
    different shapes and bit widths, each hinting its successor (the tail L2
    prefetch runs for every CTA), replayed twice -- outputs bit-identical to the
    oracle and to the unhinted run; also on producer-quantized activations."""
    rng = np.random.default_rng(44)
    shapes = [(1, 4096, 4096, 4, 4), (2, 11008, 4096, 2, 8), (1, 4096, 11008, 2, 8), (3, 700, 1500, 3, 6),
              (1, 12288, 4096, 8, 8)]
    lins, cases = [], []
    for m, n, k, wb, ab in shapes:
        x, wc, sb, zb = _case(rng, m, n, k, wb, ab)
        w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
        lins.append(abq.Linear(w, abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m))
        ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
        cases.append((torch.from_numpy(x).cuda(), orc.quantized_linear(ac, ab, sa, za, wc, wb, sb, zb)))
    plain = [lin(x, out_dtype=torch.float64).cpu().numpy() for lin, (x, _) in zip(lins, cases)]
    for i, lin in enumerate(lins):
        lin.prefetch_next(lins[(i + 1) % len(lins)])
    outs = [torch.empty((x.shape[0], lin.w.planes.rows), dtype=torch.float64, device="cuda")
            for lin, (x, _) in zip(lins, cases)]
    for _ in range(2):
        for lin, (x, _), y in zip(lins, cases, outs):
            lin(x, out=y)
    torch.cuda.synchronize()
    for i, ((_, want), y) in enumerate(zip(cases, outs)):
        assert np.array_equal(y.cpu().numpy(), want), shapes[i]
        assert np.array_equal(plain[i], want), shapes[i]
    # producer-quantized activations (abq_linear_qact) with the hint set
    spec = abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN)
    xq = torch.from_numpy((rng.standard_normal((1, 4096))).astype(np.float16)).cuda()
    g = torch.ones(4096, dtype=torch.float16, device="cuda")
    qa = abq.QAct(1, 4096, spec)
    h = torch.empty((1, 4096), dtype=torch.float16, device="cuda")
    abq.rmsnorm_quant(xq, g, 1e-6, spec, out=qa, y_out=h)
    y_q = lins[0](qa, out_dtype=torch.float64).cpu().numpy()
    lins[0].prefetch_next(None)
    y_f = lins[0](h, out_dtype=torch.float64).cpu().numpy()
    assert np.array_equal(y_q, y_f)
