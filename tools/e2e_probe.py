"""Where the end-to-end step (GraphedLinear: H2D x, engine, D2H y) spends its
time: graphs of copies only, kernel only, and both, replayed back to back."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_08554_b200 as abq  # noqa: E402

m, n, k, wb, ab, _ = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2_w4a4_m1"]
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, 24)
spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
lins = [abq.Linear(w, spec, max_m=m) for w in ws]
xh = torch.from_numpy(x_np).pin_memory()
yh = torch.empty((m, n), dtype=torch.float16).pin_memory()
xd = torch.empty((m, k), dtype=torch.float16, device="cuda")
yd = torch.empty((m, n), dtype=torch.float16, device="cuda")


def graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.current_stream().wait_stream(s)
    gs = []
    for i in range(24):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(i)
        gs.append(g)
    return gs


def timeit(gs, reps=480):
    for g in gs:
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gs[0].replay()
    e0.record()
    for i in range(reps):
        gs[i % len(gs)].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def copies(i):
    xd.copy_(xh, non_blocking=True)
    yh.copy_(yd, non_blocking=True)


def kernel(i):
    lins[i](xd, out=yd)


def both(i):
    xd.copy_(xh, non_blocking=True)
    lins[i](xd, out=yd)
    yh.copy_(yd, non_blocking=True)


def h2d(i):
    xd.copy_(xh, non_blocking=True)


def d2h(i):
    yh.copy_(yd, non_blocking=True)


for name, fn in (("H2D only", h2d), ("D2H only", d2h), ("copies", copies), ("kernel", kernel), ("all", both)):
    print(f"{name:10s} {timeit(graph(fn)):7.2f} us per step (one graph per step)")
# one graph of 24 steps
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(24):
        both(i)
print(f"{'all x24':10s} {timeit([g], 20) / 24:7.2f} us per step (24 steps per graph)")

# zero-copy output: the GEMV epilogue writes y straight into the pinned host
# buffer (UVA-mapped), no D2H copy node
import ctypes as C  # noqa: E402
L = abq._lib
lib = L.lib()
yh_ptr = yh.data_ptr()


def both_zc(i):
    xd.copy_(xh, non_blocking=True)
    lin = lins[i]
    abq.api._check(lib.abq_linear(xd.data_ptr(), L.ABQ_F16, m, k, C.byref(lin._sc), C.byref(lin._wc), yh_ptr,
                                  L.ABQ_OUT_F16, lin.ws.data_ptr(), lin.ws_bytes, lin.err.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream))


print(f"{'h2d+zc':10s} {timeit(graph(both_zc)):7.2f} us per step (one graph per step, y written to pinned host)")
torch.cuda.synchronize()
want = lins[0](torch.from_numpy(x_np).cuda()).cpu()
both_zc(0)
torch.cuda.synchronize()
print("zero-copy output equals the device output:", bool(torch.equal(yh, want)))
