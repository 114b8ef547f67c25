timeout 600 python tools/gemm_sched_sweep.py cfg3_w4a8_o_m128 cfg3_w4a8_down_m128
for s in classic stream_k; do for w in cfg3_w4a8_o_m128 cfg3_w4a8_down_m128; do echo "== trace $w $s"; timeout 300 python tools/trace_gemm.py $w f16 $s 2>&1 | grep -v Warn | sed -n 1,12p; done; done
