#!/usr/bin/env python
"""bench.py -- ABQ-LLM bit-plane quantized linear on B200 (driver contract).

One step = one pass of the hot path over one batch:
    fp16 activations (resident in HBM)
      -> K1 ReQuant + BitPacking (per-token asymmetric, FP64, round-half-away)
      -> K2 plane GEMV: sum_{s,t} 2^(s+t) popc(A_s & W_t) over the packed weights
      -> K4 fused zero-point correction + dequant -> fp16 output
on the BASELINE.json configs[1] workload (LLaMA-7B up_proj, K=4096 N=11008,
W4A4, M=1 decode).  value = packed weight bytes / step time (GB/s, the
metric's HBM GB/s on packed weight bytes), whole job over all ranks.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload NAME] [--sweep]

L2 hygiene: each step reads a different copy of the packed weights, rotating
over enough copies to exceed 4x the L2 size, so every step streams its
weights from HBM.  Steps are replayed from a CUDA graph (launch overhead is
not part of a serving step), timed with CUDA events on the launching stream,
max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]

# name -> (m, n, k, w_bits, a_bits, description)
WORKLOADS = {
    "cfg2_w4a4_m1": (1, 11008, 4096, 4, 4, "cfg2 W4A4 GEMV M=1 K=4096 N=11008 (LLaMA-7B up_proj)"),
    "cfg2_w8a8_m1": (1, 11008, 4096, 8, 8, "cfg2 W8A8 GEMV M=1 K=4096 N=11008 (LLaMA-7B up_proj)"),
    "cfg1_w2a8": (1, 4096, 4096, 2, 8, "cfg1 W2A8 GEMV M=1 K=N=4096 (LLaMA-7B q_proj)"),
}
for _m in (4, 8, 16, 128):
    for _w in (4, 8):
        WORKLOADS[f"cfg2_w{_w}a{_w}_m{_m}"] = (
            _m, 11008, 4096, _w, _w, f"cfg2 W{_w}A{_w} M={_m} K=4096 N=11008 (LLaMA-7B up_proj)")


def packed_bytes(n, k, w_bits):
    return w_bits * n * ((k + 63) // 64) * 8


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        window = [p for t, p in self.samples if t0 - 0.05 <= t <= t1 + 0.05] or [p for _, p in self.samples]
        if not window:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = sorted(float(p[0]) for p in window if p[0].replace(".", "").isdigit())
        mx = max((float(p[1]) for p in window if p[1].replace(".", "").isdigit()), default=None)
        reasons = sorted({self.NAMES[i] for p in window for i in range(4) if p[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(window)}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


def ncu_traffic(kernel_key: str):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    v = d.get(kernel_key)
    return None if v is None else v.get("dram_bytes_per_launch")


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU implementation on the host cores
# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle.oracle import RefOracle
    m, n, k, wb, ab, desc = WORKLOADS[args.workload]
    rng = np.random.default_rng(42)
    x = rng.standard_normal((m, k)).astype(np.float16).astype(np.float64)
    wc = rng.integers(0, 1 << wb, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wb, n).astype(np.int32)
    cores = os.cpu_count() or 1
    kind = "reference" if RefOracle.available() else None
    if kind is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    ref = RefOracle()
    run = ref.linear(wc, wb, sb, zb, threads=cores)
    out = np.zeros((m, n))
    for _ in range(max(1, args.warmup)):
        run(x, ab, out)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run(x, ab, out)
    dt = (time.perf_counter() - t0) / args.steps
    gbs = packed_bytes(n, k, wb) / dt / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": desc, "m": m, "n": n, "k": k, "w_bits": wb, "a_bits": ab},
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": cores, "kind": kind,
                         "sample": f"full workload per step: reference quantize+bitpack+code_rowsums+"
                                   f"gemm_arbitrary(default_tile)+zero_point_correct+dequant, weights "
                                   f"pre-packed, output channels split over {cores} threads"},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline_sample(m, n, k, wb, ab, budget_s=8.0):
    """The reference step timed on 1 host thread (the reference's own thread
    count at M<=64, gemm.hpp:88-92) over a bounded sample of the workload."""
    from oracle.oracle import RefOracle
    rng = np.random.default_rng(42)
    x = rng.standard_normal((m, k)).astype(np.float16).astype(np.float64)
    wc = rng.integers(0, 1 << wb, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wb, n).astype(np.int32)
    if not RefOracle.available():
        return None
    run = RefOracle().linear(wc, wb, sb, zb, threads=1)
    out = np.zeros((m, n))
    run(x, ab, out)
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        run(x, ab, out)
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(packed_bytes(n, k, wb) / dt / 1e9, 4), "unit": "GB/s", "cores": 1,
            "kind": "reference",
            "sample": f"{reps} full-workload reference steps ({dt * 1e3:.2f} ms each) in {budget_s:.0f} s: "
                      "quantize+bitpack+gemm_arbitrary(default_tile)+zero_point_correct+dequant, "
                      "weights pre-packed, 1 thread (reference uses ceil(M/64) threads)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def build_layer(abq, torch, m, n, k, wb, ab, copies, seed=42):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((m, k)).astype(np.float16)
    wc = rng.integers(0, 1 << wb, (n, k), dtype=np.uint8)
    sb = rng.uniform(1e-3, 1e-2, n)
    zb = rng.integers(0, 1 << wb, n).astype(np.int32)
    base = abq.PackedWeights.from_planes(abq.bitpack(wc, wb), sb, zb)
    ws = [base] + [base.copy() for _ in range(copies - 1)]
    return x, wc, sb, zb, ws


def time_graph(torch, body, copies, steps, warmup, world):
    """Capture `copies` steps (one per weight copy) in a CUDA graph and replay
    until exactly `steps` steps ran; returns total device ms (max over ranks)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(copies):
            body(i)
    torch.cuda.current_stream().wait_stream(s)
    g_full = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_full):
        for i in range(copies):
            body(i)
    rem = steps % copies
    g_rem = None
    if rem:
        g_rem = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_rem):
            for i in range(rem):
                body(i)
    for _ in range(max(1, -(-warmup // copies))):
        g_full.replay()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    e0.record()
    for _ in range(steps // copies):
        g_full.replay()
    if g_rem is not None:
        g_rem.replay()
    e1.record()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    return ms, (t_wall0, t_wall1)


def run_ours(args, world, rank, local):
    import torch

    import paper_2408_08554_b200 as abq
    m, n, k, wb, ab, desc = WORKLOADS[args.workload]
    # column-parallel sharding, weak scaling: the layer has
    # world x N output channels and rank r owns channels [r*N, (r+1)*N) -- the
    # workload's N per GPU at every GPU count.  No data-path collective; the
    # output all-gather (where a layer's output must be reassembled) is timed
    # as a separate leg below.
    n_full = n * world
    wbytes_full = packed_bytes(n_full, k, wb)
    wbytes = packed_bytes(n, k, wb)
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    copies = int(min(256, max(2, math.ceil(4 * l2 / wbytes))))
    # every rank draws the same activations (seeded) and its own weight shard
    x_np, wc, sb, zb, ws = build_layer(abq, torch, m, n, k, wb, ab, 1, seed=42 + rank)
    x_np = np.random.default_rng(42).standard_normal((m, k)).astype(np.float16)
    shard = ws[0]
    if args.variant != "auto":
        abq.api.set_gemv_variant(args.variant)
    weights = [shard] + [shard.copy() for _ in range(copies - 1)]
    if args.variant == "popc":  # keep only the ABQP planes resident
        for w in weights:
            w.frag = None
            w.tc = None
    spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
    lins = [abq.Linear(w, spec, max_m=m) for w in weights]
    if not args.no_prefetch_next:  # the layer sequence is known: hint each layer's successor
        for i, lin in enumerate(lins):
            lin.prefetch_next(lins[(i + 1) % len(lins)])
    x = torch.from_numpy(x_np).cuda()
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")

    # ---- parity check of this exact workload against the oracle (rank 0's shard)
    parity = None
    if rank == 0 and not args.no_check:
        from oracle.oracle import COracle
        orc = COracle()
        y64 = lins[0](x, out_dtype=torch.float64).cpu().numpy()
        ac, sa, za = orc.quantize(x_np.astype(np.float64), ab, 0, 2)
        want = orc.quantized_linear(ac, ab, sa, za, wc, wb, sb, zb)
        y16 = lins[0](x, out_dtype=torch.float16).cpu().numpy()
        parity = bool(np.array_equal(y64, want) and np.array_equal(y16, want.astype(np.float16)))
        if not parity:
            raise SystemExit("bench: engine output differs from the oracle -- refusing to report")

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = abq.launch_count()

    # ---- headline: full step (K1 + K2/K4), weights rotated past L2
    ms, (tw0, tw1) = time_graph(torch, lambda i: lins[i](x, out=y, check=False), copies, args.steps,
                                args.warmup, world)
    step_launches = (abq.launch_count() - launches0)
    clocks.stop()
    clk = clocks.summary(tw0, tw1)
    ms_per_step = ms / args.steps
    value = wbytes_full / (ms_per_step * 1e-3) / 1e9  # whole-job bytes (all ranks) per step time

    # graph capture recorded (copies + rem + warm) * launches-per-step; launches per step:
    per_step = 0
    a0 = abq.launch_count()
    lins[0](x, out=y, check=False)
    per_step = abq.launch_count() - a0
    gpu_launches = per_step * args.steps

    # ---- dominant kernel: with the fused single-launch path the step IS the
    # kernel (timed above with CUDA events on its stream); otherwise time the
    # GEMV + fused-epilogue kernel alone, back to back, on the same rotation.
    fused = per_step == 1
    if fused:
        kernel_us = ms_per_step * 1e3
        kernel_name = "gemv_dec_kernel (ReQuant prologue + tensor-pipe plane GEMV + epilogue)"
    else:
        a_planes, sa, za, ra = abq.api.quant_pack_act(x, spec)
        kms, _ = time_graph(torch, lambda i: abq.linear_planes(a_planes, sa, za, ra, weights[i], out=y),
                            copies, args.steps, args.warmup, world)
        kernel_us = kms * 1e3 / args.steps
        kernel_name = "gemv_popc_kernel (AND+popcount plane GEMV + epilogue)"
    peak, peak_kind, _ = measured_peaks()
    achieved = wbytes / (kernel_us * 1e-6) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(args.workload),
                "kernel": kernel_name, "kernel_us": round(kernel_us, 3),
                "algorithmic_bytes_per_launch": wbytes, "peak_kind": f"of {peak_kind}",
                "kernel_share_of_step": round(kernel_us / (ms_per_step * 1e3), 3)}

    # ---- end to end through the public API with host buffers (GraphedLinear:
    # H2D x from pinned host, engine, D2H y into pinned host, every step)
    e2e = None
    if True:
        gl = [abq.GraphedLinear(lins[i], m) for i in range(min(copies, 64))]
        for g in gl:
            g.x_host.copy_(torch.from_numpy(x_np))
        for i in range(args.warmup):
            gl[i % len(gl)].step()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            gl[i % len(gl)].step()
        e1.record()
        torch.cuda.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1), world) / args.steps
        # eager (per-call Python API, no graph) for reference
        t0 = time.perf_counter()
        eager_steps = min(args.steps, 2000)
        xh = gl[0].x_host
        yh = gl[0].y_host
        xd = torch.empty_like(gl[0].x_dev)
        for i in range(eager_steps):
            xd.copy_(xh, non_blocking=True)
            lins[i % copies](xd, out=y, check=False)
            yh.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
        eager_ms = (time.perf_counter() - t0) * 1e3 / eager_steps
        e2e = {"value": round(wbytes_full / (e_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
               "h2d_bytes_per_step": gl[0].h2d_bytes, "d2h_bytes_per_step": gl[0].d2h_bytes,
               "ms_per_step": round(e_ms, 5), "api": "abq.GraphedLinear.step()",
               "eager_api_ms_per_step": round(eager_ms, 5)}

    # ---- reassembly leg (N > 1): the same step followed by the NCCL all-gather
    # of the fp16 output slices over NVLink (sharded.gather_columns), captured in
    # the same kind of CUDA graph; reported beside the compute-only headline.
    gather = None
    if world > 1:
        import torch.distributed as dist
        buf = torch.empty((world, m, n), dtype=torch.float16, device="cuda")

        def step_gather(i):
            lins[i](x, out=y, check=False)
            dist.all_gather_into_tensor(buf, y)
        try:
            g_ms, _ = time_graph(torch, step_gather, copies, args.steps, args.warmup, world)
            how = "CUDA graph (engine step + ncclAllGather)"
        except Exception as exc:  # graph capture of the collective unavailable: eager loop
            torch.cuda.synchronize()
            barrier(world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(args.steps):
                step_gather(i % copies)
            e1.record()
            torch.cuda.synchronize()
            g_ms = max_over_ranks(e0.elapsed_time(e1), world)
            how = f"eager loop ({type(exc).__name__} capturing the collective)"
        g_step = g_ms / args.steps
        gather = {"ms_per_step": round(g_step, 6), "value": round(wbytes_full / (g_step * 1e-3) / 1e9, 1),
                  "unit": "GB/s", "gather_bytes_per_rank": m * n * 2, "timing": how}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_sample(m, n_full, k, wb, ab, budget_s=args.cpu_seconds)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 6),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic",
        "config": {"workload": desc, "m": m, "n": n_full, "n_per_gpu": n, "k": k, "w_bits": wb, "a_bits": ab,
                   "parallelism": f"N-sharded x{world} (column-parallel)" if world > 1 else "single",
                   "l2": f"rotating {copies} packed-weight copies ({copies * wbytes / 1e6:.0f} MB > 4x L2)",
                   "step": "fp16 x -> ReQuant+BitPack -> plane GEMV -> zero-point+dequant -> fp16 y",
                   "graph": "CUDA graph replay",
                   "prefetch_next": not args.no_prefetch_next},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches,
        "launches_per_step": per_step, "clocks": clk, "parity": "bit-exact vs oracle" if parity else None,
        "allgather": gather,
    }
    if args.sweep and rank == 0:
        line["sweep"] = sweep(abq, torch, world)
    if rank == 0:
        print(json.dumps(line))


def sweep(abq, torch, world):
    """kernel-level table over the BASELINE configs (not the headline)."""
    rows = []
    for name, (m, n, k, wb, ab, desc) in WORKLOADS.items():
        x_np, wc, sb, zb, _ = build_layer(abq, torch, m, n, k, wb, ab, 1)
        wbytes = packed_bytes(n, k, wb)
        l2 = torch.cuda.get_device_properties(0).L2_cache_size
        copies = int(min(128, max(2, math.ceil(4 * l2 / wbytes))))
        _, _, _, _, ws = build_layer(abq, torch, m, n, k, wb, ab, copies)
        spec = abq.QuantSpec(bits=ab, granularity=abq.api.PER_TOKEN)
        lins = [abq.Linear(w, spec, max_m=m) for w in ws]
        x = torch.from_numpy(x_np).cuda()
        y = torch.empty((m, n), dtype=torch.float16, device="cuda")
        steps = 400
        ms, _ = time_graph(torch, lambda i: lins[i](x, out=y, check=False), copies, steps, 20, world)
        a_planes, sa, za, ra = abq.api.quant_pack_act(x, spec)
        kms, _ = time_graph(torch, lambda i: abq.linear_planes(a_planes, sa, za, ra, ws[i], out=y),
                            copies, steps, 20, world)
        step_us, kern_us = ms * 1e3 / steps, kms * 1e3 / steps
        row = {"workload": name, "step_us": round(step_us, 3), "kernel_us": round(kern_us, 3),
               "kernel_GBps": round(wbytes / kern_us / 1e3, 1), "TOPS": round(2 * m * n * k / step_us / 1e6, 2)}
        if m >= 16 and (ab, wb) in ((4, 4), (8, 8), (8, 2), (8, 4), (4, 8), (2, 2)):
            # b1 tensor-core (mma.sync .b1 and.popc) plane GEMM, the BTC alternative
            bsteps = 40
            bms, _ = time_graph(torch, lambda i: abq.gemm_btc(a_planes, ws[i].planes), copies, bsteps, 3, world)
            row["btc_b1_gemm_us"] = round(bms * 1e3 / bsteps, 3)
        if m >= 8:
            # cuBLAS fp16 comparator at the same shape (weights rotated past L2)
            wf = [torch.randn((n, k), dtype=torch.float16, device="cuda") for _ in range(
                max(2, math.ceil(4 * l2 / (n * k * 2))))]
            xf = torch.randn((m, k), dtype=torch.float16, device="cuda")
            yf = torch.empty((m, n), dtype=torch.float16, device="cuda")
            cms, _ = time_graph(torch, lambda i: torch.matmul(xf, wf[i].t(), out=yf), len(wf), steps, 20,
                                world)
            row["cublas_fp16_us"] = round(cms * 1e3 / steps, 3)
        rows.append(row)
        del lins, ws
        torch.cuda.empty_cache()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="abq", choices=["abq", "reference"])
    ap.add_argument("--workload", default="cfg2_w4a4_m1", choices=sorted(WORKLOADS))
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-prefetch-next", action="store_true",
                    help="do not give each layer its successor as an L2 prefetch hint")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--variant", default="auto", choices=["auto", "popc", "recomb"],
                    help="decode GEMV: auto | popc (AND+popcount) | recomb (planes on the int8 tensor pipe)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup(args)
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
