"""Device-side timeline of back-to-back engine linears inside one CUDA graph
(globaltimer stamps per CTA): kernel span and the gap between consecutive
kernels.  Usage: python tools/trace_graph.py [workload] [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_08554_b200 as abq  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2_w4a4_m1"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 6
m, n, k, wb, ab, desc = bench.WORKLOADS[name]
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, L)
spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
lins = [abq.Linear(w, spec, max_m=m) for w in ws]
x = torch.from_numpy(x_np).cuda()
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
bufs = [torch.zeros(16 * 4096, dtype=torch.int64, device="cuda") for _ in range(L)]
lib = abq._lib.lib()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(L):
        lins[i](x, out=y, check=False)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(L):
        lib.abq_set_trace_buffer(bufs[i].data_ptr())
        lins[i](x, out=y, check=False)
lib.abq_set_trace_buffer(None)
for _ in range(3):
    for b in bufs:
        b.zero_()
    g.replay()
torch.cuda.synchronize()
spans = []
for b in bufs:
    t = b.view(-1, 16).cpu().numpy().astype(np.int64)
    t = t[t[:, 8] > 0]
    spans.append((t[:, 8].min(), t[:, 9].max()))
print(f"{name}: {L} graph-captured launches")
for i, (a, e) in enumerate(spans):
    gap = "" if i == 0 else f"  gap from previous end {(a - spans[i - 1][1]) / 1e3:6.2f} us"
    print(f"  launch {i}: span {(e - a) / 1e3:6.2f} us{gap}")
print(f"  first start -> last end {(spans[-1][1] - spans[0][0]) / 1e3:.2f} us = "
      f"{(spans[-1][1] - spans[0][0]) / 1e3 / L:.2f} us per launch")
