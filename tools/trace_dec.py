"""Device-side timeline of the serving decode GEMV (gemv_dec_kernel) inside a
CUDA graph of back-to-back layers, from the TRACE build of the library
(make -C paper_2408_08554_b200/csrc TRACE=1; this script sets ABQ_LIB to it).
Per launch: the CTA span (globaltimer), the gap to the previous launch, the
CTA start skew, and per-CTA phase marks (SM clock, median over CTAs, us from
CTA start): set-up done, griddepcontrol.wait returned, range (min/max) done,
step / zero point done, codes done (prologue end), main loop done, epilogue done.
Usage: python tools/trace_dec.py [workload] [launches]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("ABQ_LIB", os.path.join(ROOT, "paper_2408_08554_b200", "libabq_cuda_trace.so"))
sys.path.insert(0, ROOT)
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
x = torch.from_numpy(x_np).cuda()
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
bufs = [torch.zeros(64 * 4096, dtype=torch.int64, device="cuda") for _ in range(L)]
lib = abq._lib.lib()
for kv in os.environ.get("ABQ_TUNE", "").split(","):
    if kv:
        key, val = kv.split("=")
        lib.abq_set_tuning(key.encode(), int(val))
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
if len(rows[0]) == 0:
    raise SystemExit("no stamps: is ABQ_LIB the trace build (make TRACE=1)?")
print(f"{name} ({desc}): {L} graph-captured launches, {len(rows[0])} CTAs")
prev_end = None
names = ("setup", "wait", "range", "step", "codes", "main", "epilogue")
for i, t in enumerate(rows):
    a, e = t[:, 8].min(), t[:, 9].max()
    gap = "" if prev_end is None else f"  start - previous end {(a - prev_end) / 1e3:6.2f} us"
    marks = [np.median(t[:, c] - t[:, 0]) / ghz / 1e3 for c in range(1, 8)]
    print(f"  launch {i:2d}: span {(e - a) / 1e3:6.2f} us{gap}  (CTA start skew {(t[:, 8].max() - a) / 1e3:5.2f} us)")
    print("             " + ", ".join(f"{nm} {v:.2f}" for nm, v in zip(names, marks)))
    sp = [np.median(t[:, c] - t[:, 3]) / ghz / 1e3 for c in (10, 11, 4)]
    print("             step phase (us after range): reductions %.2f, group_params %.2f, stored %.2f" % tuple(sp))
    d = [np.median(t[:, c] - t[:, 5]) / ghz / 1e3 for c in (16, 17, 18, 19, 20)]
    we = (t[:, 24:40] - t[:, 5:6]) / ghz / 1e3
    print("             main loop (warp 0, us after codes): start %.2f, first data %.2f, first fold %.2f, loop end %.2f, flush end %.2f;"
          " warp ends: min %.2f median %.2f max %.2f" % (*d, np.median(we.min(1)), np.median(np.median(we, 1)), np.median(we.max(1))))
    prev_end = e
first, last = rows[0][:, 8].min(), rows[-1][:, 9].max()
print(f"  first start -> last end {(last - first) / 1e3:.2f} us = {(last - first) / 1e3 / L:.3f} us per launch")
