"""Phase timing (per CTA, SM clock) of the tcgen05 prefill GEMM: time to the
first MMA, MMA issue progress every 8 k-blocks, epilogue, plus the device span
of the launch (globaltimer).  Usage: python tools/trace_gemm.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_08554_b200 as abq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_w4a4_m128"
m, n, k, wb, ab, desc = bench.WORKLOADS[name]
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, 2)
spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
lins = [abq.Linear(w, spec, max_m=m) for w in ws]
x = torch.from_numpy(x_np).cuda()
odt = {"f16": torch.float16, "f32": torch.float32, "f64": torch.float64}[sys.argv[2] if len(sys.argv) > 2 else "f16"]
y = torch.empty((m, n), dtype=odt, device="cuda")
buf = torch.zeros(64 * 4096, dtype=torch.int64, device="cuda")
for _ in range(3):
    lins[0](x, out=y, check=False)
torch.cuda.synchronize()
lib = abq._lib.lib()
for kv in os.environ.get("ABQ_TUNE", "").split(","):
    if kv:
        key, val = kv.split("=")
        lib.abq_set_tuning(key.encode(), int(val))
if len(sys.argv) > 3:
    abq.api.set_gemm_schedule(sys.argv[3])
    for _ in range(3):
        lins[0](x, out=y, check=False)
    torch.cuda.synchronize()
lib.abq_set_trace_buffer(buf.data_ptr())
lins[1](x, out=y, check=False)
torch.cuda.synchronize()
lib.abq_set_trace_buffer(None)
t = buf.view(-1, 64).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
ghz = 1.965


def us(a):
    return a / ghz / 1e3


print(f"{name}: {len(t)} CTAs")
print(f"  first MMA issued         median {np.median(us(t[:, 32] - t[:, 0])):7.2f} us after CTA start")
print(f"  last MMA issued          median {np.median(us(t[:, 3] - t[:, 0])):7.2f} us")
print(f"  epilogue start (done)    median {np.median(us(t[:, 4] - t[:, 0])):7.2f} us")
con, fin = t[:, 10] > 0, t[:, 11] > 0
if con.any():  # stream-K
    print(f"  stream-K: units/CTA {np.unique(t[:, 12] >> 32)}, contributors/finish {np.unique((t[fin, 12] >> 8) & 255)}")
    print(f"  partial published        median {np.median(us(t[con, 10] - t[con, 0])):7.2f} us")
    print(f"  finisher wait done       median {np.median(us(t[fin, 11] - t[fin, 0])):7.2f} us  max {us(t[fin, 11] - t[fin, 0]).max():7.2f}")
print(f"  tid0 epilogue math done median {np.median(us(t[:, 6] - t[:, 0])):7.2f} us; after barrier {np.median(us(t[:, 7] - t[:, 0])):7.2f}")
print(f"  CTA end                  median {np.median(us(t[:, 5] - t[:, 0])):7.2f} us  max {us(t[:, 5] - t[:, 0]).max():7.2f}")
print(f"  launch span (globaltimer) {(t[:, 9].max() - t[:, 8].min()) / 1e3:7.2f} us; CTA start skew "
      f"{(t[:, 8].max() - t[:, 8].min()) / 1e3:6.2f} us")

c0 = t[0]
print("  CTA 0 per k-block (us after start): widened / MMA issued / producer refill issued (stage kb+S)")
for kb in range(16):
    w, mm, pr = c0[16 + kb], c0[32 + kb], c0[48 + kb]
    f = lambda v: "%6.2f" % us(v - c0[0]) if v > 0 else "   -  "
    print("   kb %2d: %s %s %s" % (kb, f(w), f(mm), f(pr)))
