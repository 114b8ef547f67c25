"""Phase timing (SM clock cycles, per CTA) of the fused decode GEMV:
prologue (wait for ReQuant codes), main loop, epilogue.
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
x_np, wc, sb, zb, ws = bench.build_layer(abq, torch, m, n, k, wb, ab, 1)
lin = abq.Linear(ws[0], abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN), max_m=m)
x = torch.from_numpy(x_np).cuda()
buf = torch.zeros(8 * 148 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    lin(x, check=False)
abq._lib.lib().abq_set_trace_buffer(buf.data_ptr())
lin(x, check=False)
torch.cuda.synchronize()
abq._lib.lib().abq_set_trace_buffer(None)
t = buf.view(-1, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
ghz = 1.965
def stat(a, lab):
    print(f"  {lab:28s} median {np.median(a) / ghz / 1e3:6.2f} us  max {a.max() / ghz / 1e3:6.2f} us")
print(f"{name}: {len(t)} CTAs, local row-tiles/CTA median {np.median(t[:, 4]):.0f}")
stat(t[:, 1] - t[:, 0], "prologue (wait + act copy)")
stat(t[:, 2] - t[:, 1], "main loop (first warp done)")
stat(t[:, 6] - t[:, 1], "main loop (last warp done)")
stat(t[:, 5] - t[:, 6], "owned-tile epilogue")
stat(t[:, 6] - t[:, 0], "start -> last warp done")
stat(t[:, 3] - t[:, 5], "split-tile atomics")
