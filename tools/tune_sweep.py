"""Engine-schedule autotune (abq.autotune_linear) over LLaMA-like prefill and
decode shapes, W4A4 per-token; prints BenchRecord CSV (tune.hpp:94-105 schema).
Usage (GPU): python tools/tune_sweep.py > profiles/r01_tune_sweep.csv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_08554_b200 as abq  # noqa: E402

SHAPES = [(1, 11008, 4096), (16, 11008, 4096), (128, 11008, 4096), (128, 4096, 4096), (128, 4096, 11008),
          (128, 2048, 4096), (128, 1024, 11008), (256, 4096, 4096), (64, 1024, 4096)]
print(abq.BenchRecord.csv_header() + ",best")
rng = np.random.default_rng(0)
for m, n, k in SHAPES:
    wc = rng.integers(0, 16, (n, k), dtype=np.uint8)
    w = abq.PackedWeights.from_planes(abq.bitpack(wc, 4), rng.uniform(1e-3, 1e-2, n),
                                      rng.integers(0, 16, n).astype(np.int32))
    lin = abq.Linear(w, abq.QuantSpec(bits=4, granularity=abq.api.PER_TOKEN), max_m=m)
    x = torch.from_numpy((rng.standard_normal((m, k)) * 2).astype(np.float16)).cuda()
    res = abq.autotune_linear(lin, x, trials=21)
    for r in res.records:
        print(r.csv_row() + ("," + res.best if r.config_id == res.best else ","))
    abq.set_gemv_variant("auto")
    abq.set_gemm_schedule("auto")
    sys.stdout.flush()
