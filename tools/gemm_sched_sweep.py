"""Step time of M >= 9 workloads under each prefill GEMM schedule (auto /
classic / stream_k), L2-cold rotation, CUDA-graph replay (bench.measure_part).
Usage: python tools/gemm_sched_sweep.py workload [workload ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_08554_b200 as abq  # noqa: E402

peaks, kind = bench.measured_peaks()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for name in sys.argv[1:]:
    for sched in ("auto", "classic", "stream_k"):
        abq.api.set_gemm_schedule(sched)
        r = bench.measure_part(abq, torch, name, 1, 200, 10, l2, peaks, kind)
        print(f"{name:24s} {sched:9s} {r['step_us']:8.2f} us  cuBLAS {r.get('cublas_fp16_us')} us", flush=True)
    abq.api.set_gemm_schedule("auto")
