O=gpurun_out; T=${1:-gm}
for w in cfg2_w4a4_m128 cfg2_w8a8_m128; do for s in classic stream_k; do echo "== $w $s"; timeout 120 python tools/trace_gemm.py $w f16 $s 2>&1 | head -12; done; done > $O/${T}_trace.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 8 --csv python bench.py --workload cfg2_w4a4_m128 --steps 20 --warmup 3 --no-parts --no-cpu --no-check > $O/${T}_launches.csv 2>&1
