"""One small invocation of every engine kernel family (for compute-sanitizer
memcheck / racecheck / synccheck, tools/gpu_sanitize.sh), each checked against
the oracle: decode GEMV (fused ReQuant, ring refill, ReQuant-kernel + PDL,
producer-fused codes), tcgen05 GEMM (classic + stream-K), AND+popcount,
quantizer / bitpack kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_08554_b200 as abq  # noqa: E402
from oracle.oracle import COracle, exact_linear  # noqa: E402

orc = COracle()
rng = np.random.default_rng(0)
fails = 0


def case(name, m, n, k, wb, ab, sched=None, x_dtype=np.float16):
    global fails
    wc = rng.integers(0, 1 << wb, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wb, n).astype(np.int32)
    x = rng.standard_normal((m, k)).astype(x_dtype)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
    spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
    if sched:
        abq.api.set_gemm_schedule(sched)
    y = abq.Linear(w, spec, max_m=m)(torch.from_numpy(x).cuda(), out_dtype=torch.float64, check=True)
    abq.api.set_gemm_schedule("auto")
    ac, sa, za = orc.quantize(x.astype(np.float64), ab, 0, 2)
    ok = np.array_equal(y.cpu().numpy(), exact_linear(ac, sa, za, wc, sb, zb))
    fails += not ok
    print(f"{'ok  ' if ok else 'FAIL'} {name}", flush=True)


case("decode W4A4 M=1 (fused ReQuant)", 1, 2048, 4096, 4, 4)
case("decode W2A8 M=1 K=11008", 1, 1024, 11008, 2, 8)
case("decode W8A8 M=1 ring refill", 1, 4096, 4096, 8, 8)
case("decode W3A5 M=3 (widened slices)", 3, 600, 2048, 3, 5)
case("decode W4A4 M=8 (ReQuant kernel + PDL)", 8, 1024, 4096, 4, 4)
case("decode fp32 input M=2", 2, 512, 1024, 4, 8, x_dtype=np.float32)
case("tcgen05 GEMM W4A4 M=128 classic", 128, 1024, 4096, 4, 4, sched="classic")
case("tcgen05 GEMM W4A4 M=128 stream-K", 128, 1024, 4096, 4, 4, sched="stream_k")
case("tcgen05 GEMM W8A8 M=64", 64, 512, 2048, 8, 8)
case("tcgen05 GEMM W2A4 M=300", 300, 384, 1024, 2, 4)
# producer-fused ReQuant -> decode GEMV
spec = abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN)
x = torch.from_numpy(rng.standard_normal((2, 4096)).astype(np.float16)).cuda()
g = torch.ones(4096, dtype=torch.float16, device="cuda")
yn = torch.empty_like(x)
qa = abq.rmsnorm_quant(x, g, 1e-6, spec, y_out=yn, check=True)
wc = rng.integers(0, 16, (1024, 4096), dtype=np.uint8)
sb, zb = rng.uniform(1e-3, 1e-2, 1024), rng.integers(0, 16, 1024).astype(np.int32)
w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), sb, zb)
out = abq.Linear(w, spec, max_m=2)(qa, out_dtype=torch.float64).cpu().numpy()
ac, sa, za = orc.quantize(yn.cpu().numpy().astype(np.float64), 4, 0, 2)
ok = np.array_equal(out, exact_linear(ac, sa, za, wc, sb, zb))
fails += not ok
print(f"{'ok  ' if ok else 'FAIL'} producer rmsnorm_quant -> linear_qact", flush=True)
up = torch.from_numpy(rng.standard_normal((2, 4096)).astype(np.float16)).cuda()
abq.silu_mul_quant(x, up, spec, check=True)
# API path: AND+popcount, bitpack / unpack / quantize / bmma / zero-point kernels
a = rng.integers(0, 16, (5, 700), dtype=np.uint8)
b = rng.integers(0, 8, (33, 700), dtype=np.uint8)
pa, pb = abq.bitpack(a, 4), abq.bitpack(b, 3)
got = abq.gemm_arbitrary(pa, pb, abq.default_tile(4, 3)).cpu().numpy()
ok = np.array_equal(got, a.astype(np.int64) @ b.astype(np.int64).T) and np.array_equal(abq.unpack(pa).cpu().numpy(), a)
fails += not ok
print(f"{'ok  ' if ok else 'FAIL'} AND+popcount gemm_arbitrary / bitpack / unpack", flush=True)
qt = abq.quantize(torch.from_numpy(rng.standard_normal((4, 300))).cuda(), abq.QuantSpec(bits=5))
abq.bmma(pa, 1, pb, 2)
torch.cuda.synchronize()
print("sanitize cases done, failures:", fails)
sys.exit(1 if fails else 0)
