timeout 900 python -m pytest tests/test_gpu_gemm_tc.py tests/test_tune.py -x -q 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/gemm_sched_sweep.py cfg3_w4a8_o_m128 cfg3_w4a8_down_m128 cfg2_w4a4_m128 cfg2_w8a8_m128
echo "== trace down stream_k"; timeout 300 python tools/trace_gemm.py cfg3_w4a8_down_m128 f16 stream_k 2>&1 | grep -v Warn | sed -n 1,10p
echo "== trace o stream_k"; timeout 300 python tools/trace_gemm.py cfg3_w4a8_o_m128 f16 stream_k 2>&1 | grep -v Warn | sed -n 1,10p
