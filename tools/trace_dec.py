"""Device-side timeline of the serving decode GEMV (gemv_dec_kernel) inside a
CUDA graph of back-to-back layers: per launch, the CTA span (globaltimer), the
overlap / gap with the previous launch, and per-CTA phase times (SM clock):
start -> prologue end (ReQuant + parameters), -> last warp done with the main
loop, -> epilogue end.
Usage: python tools/trace_dec.py [workload] [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_08554_b200 as abq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_w4a4_m1"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 12
m, n, k, wb, ab, desc = bench.WORKLOADS[name]
copies = int(sys.argv[3]) if len(sys.argv) > 3 else max(L, 2)
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, copies)
spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
lins = [abq.Linear(w, spec, max_m=m) for w in ws[:copies]]
if os.environ.get("TRACE_NO_NEXT") != "1":
    for i, lin in enumerate(lins):
        lin.prefetch_next(lins[(i + 1) % len(lins)])
x = torch.from_numpy(x_np).cuda()
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
bufs = [torch.zeros(64 * 4096, dtype=torch.int64, device="cuda") for _ in range(L)]
lib = abq._lib.lib()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(L):
        lins[i % copies](x, out=y, check=False)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(L):
        lib.abq_set_trace_buffer(bufs[i].data_ptr())
        lins[i % copies](x, out=y, check=False)
lib.abq_set_trace_buffer(None)
for _ in range(3):
    for b in bufs:
        b.zero_()
    g.replay()
torch.cuda.synchronize()
ghz = 1.965
rows = []
for b in bufs:
    t = b.view(-1, 64).cpu().numpy().astype(np.int64)
    rows.append(t[t[:, 8] > 0])
print(f"{name} ({desc}): {L} graph-captured launches, {len(rows[0])} CTAs")
prev_end = None
for i, t in enumerate(rows):
    a, e = t[:, 8].min(), t[:, 9].max()
    gap = "" if prev_end is None else f"  start - previous end {(a - prev_end) / 1e3:6.2f} us"
    pro = np.median(t[:, 1] - t[:, 0]) / ghz / 1e3
    main = np.median(t[:, 2] - t[:, 1]) / ghz / 1e3
    epi = np.median(t[:, 3] - t[:, 2]) / ghz / 1e3
    ph = [np.median(t[:, c] - t[:, 0]) / ghz / 1e3 for c in (4, 5, 6, 1)]
    print("             prologue marks (us from start): wait done %.2f, min/max %.2f, step %.2f, codes %.2f" % tuple(ph))
    print(f"  launch {i:2d}: span {(e - a) / 1e3:6.2f} us{gap}   prologue {pro:5.2f}  main {main:5.2f}  epilogue {epi:5.2f} us"
          f"  (CTA start skew {(t[:, 8].max() - a) / 1e3:5.2f} us)")
    tw = t[:, 24:40].astype(float) / ghz / 1e3
    print("             main-loop slot waits per warp: median %.2f us, max %.2f us" % (np.median(tw), tw.max()))
    en = t[:, 12]
    print("             true CTA entry: first %.2f us, median %.2f, last %.2f us after previous end; entry->first stamp median %.2f us"
          % (((en.min() - prev_end) / 1e3) if prev_end else 0, ((np.median(en) - prev_end) / 1e3) if prev_end else 0,
             ((en.max() - prev_end) / 1e3) if prev_end else 0, np.median(t[:, 8] - en) / 1e3))
    prev_end = e
first, last = rows[0][:, 8].min(), rows[-1][:, 9].max()
print(f"  first start -> last end {(last - first) / 1e3:.2f} us = {(last - first) / 1e3 / L:.3f} us per launch")
