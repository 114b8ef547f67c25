timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/gemm_sched_sweep.py cfg3_w4a8_down_m128 cfg3_w2a4_down_m128 cfg3_w6a6_down_m128
echo "== trace down classic"; timeout 300 python tools/trace_gemm.py cfg3_w4a8_down_m128 f16 classic 2>&1 | grep -v Warn | sed -n 1,8p
echo "== trace down stream_k"; timeout 300 python tools/trace_gemm.py cfg3_w4a8_down_m128 f16 stream_k 2>&1 | grep -v Warn | sed -n 1,12p
