"""Phase timing (per CTA) of the fused decode GEMV: prologue, main loop,
epilogue (SM clock cycles), plus the device-side gap between two
back-to-back launches (globaltimer).
Usage: python tools/trace_gemv.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_08554_b200 as abq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_w4a4_m1"
m, n, k, wb, ab, desc = bench.WORKLOADS[name]
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, 2)
spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
lins = [abq.Linear(w, spec, max_m=m) for w in ws]
x = torch.from_numpy(x_np).cuda()
bufs = [torch.zeros(16 * 148 * 8, dtype=torch.int64, device="cuda") for _ in range(2)]
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
for _ in range(3):
    lins[0](x, out=y, check=False)
torch.cuda.synchronize()
lib = abq._lib.lib()
for i in range(2):  # two launches back to back, each with its own trace buffer
    lib.abq_set_trace_buffer(bufs[i].data_ptr())
    lins[i](x, out=y, check=False)
torch.cuda.synchronize()
lib.abq_set_trace_buffer(None)
ts = []
for b in bufs:
    t = b.view(-1, 16).cpu().numpy().astype(np.int64)
    ts.append(t[t[:, 0] > 0])
t = ts[0]
ghz = 1.965


def stat(a, lab):
    print(f"  {lab:28s} median {np.median(a) / ghz / 1e3:6.2f} us  max {a.max() / ghz / 1e3:6.2f} us")


print(f"{name}: {len(t)} CTAs, local row-tiles/CTA median {np.median(t[:, 4]):.0f}")
stat(t[:, 1] - t[:, 0], "prologue (act + params)")
stat(t[:, 7] - t[:, 0], "  start -> ring started")
if (t[:, 10] > 0).any():
    stat(t[:, 10] - t[:, 7], "  -> min/max barrier")
    stat(t[:, 11] - t[:, 10], "  -> step/zero barrier")
    stat(t[:, 12] - t[:, 11], "  -> codes + sum barrier")
    stat(t[:, 1] - t[:, 12], "  -> prologue end")
stat(t[:, 2] - t[:, 1], "main loop (first warp done)")
stat(t[:, 6] - t[:, 1], "main loop (last warp done)")
stat(t[:, 5] - t[:, 6], "owned-tile epilogue")
stat(t[:, 6] - t[:, 0], "start -> last warp done")
stat(t[:, 3] - t[:, 5], "split-tile atomics")
a, b = ts
print(f"  launch 1 span (first CTA start -> last CTA end) {(a[:, 9].max() - a[:, 8].min()) / 1e3:6.2f} us; "
      f"CTA start skew {(a[:, 8].max() - a[:, 8].min()) / 1e3:5.2f} us")
print(f"  gap launch 1 last CTA end -> launch 2 first CTA start {(b[:, 8].min() - a[:, 9].max()) / 1e3:6.2f} us")
