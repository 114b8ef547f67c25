"""Per-CTA global timeline of the serving decode GEMV in a CUDA graph of
back-to-back layers (TRACE build, globaltimer stamps): for every launch,
percentiles over CTAs of start, griddepcontrol.wait return, prologue end,
last weight unit landed (warp 0), main loop end and CTA end, in us relative to
the previous launch's last CTA end -- split into heavy (one row-tile more) and
light CTAs.  Shows which phase the step's critical path runs through.
Usage: python tools/trace_dec_cta.py [workload] [launches]"""
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
copies = max(L, 2)
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, copies)
spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
lins = [abq.Linear(w, spec, max_m=m) for w in ws[:copies]]
if os.environ.get("ABQ_NEXT", "1") == "1":
    for i, lin in enumerate(lins):
        lin.prefetch_next(lins[(i + 1) % copies])
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
rows = []
for b in bufs:
    t = b.view(-1, 64).cpu().numpy().astype(np.int64)
    rows.append(t[: (t[:, 8] > 0).sum()])
G = len(rows[0])
rowtiles = (n + 15) // 16
heavy = np.arange(G) < rowtiles % G
print(f"{name} ({desc}): {L} launches, {G} CTAs ({heavy.sum()} heavy)")
cols = (("start", 8), ("prodissued", 15), ("slot0", 41), ("waitret", 12), ("firstdata", 22), ("codes", 13),
        ("lastdata", 21), ("lastslot", 42), ("mainend", 14), ("end", 9))
prev_end = None
steps = []
for i, t in enumerate(rows):
    if prev_end is None:
        prev_end = t[:, 8].min()
    out = []
    for nm, c in cols:
        v = (t[:, c] - prev_end) / 1e3
        parts = []
        for lab, sel in (("H", heavy), ("L", ~heavy)):
            if sel.any():
                q = np.percentile(v[sel], [0, 50, 100])
                parts.append(f"{lab} {q[0]:5.2f}/{q[1]:5.2f}/{q[2]:5.2f}")
        out.append(f"{nm:10s} " + "  ".join(parts))
    end = t[:, 9].max()
    steps.append((end - prev_end) / 1e3)
    last = int(np.argmax(t[:, 9]))
    print(f" launch {i:2d}: step {(end - prev_end) / 1e3:5.2f} us; last CTA {last} ({'heavy' if heavy[last] else 'light'})"
          " [min/median/max us after previous launch end]")
    for o in out:
        print("    " + o)
    prev_end = end
print(f" median step {np.median(steps[2:]):.2f} us")
