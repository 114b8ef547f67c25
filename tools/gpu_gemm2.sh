O=gpurun_out; T=${1:-gm}
for w in cfg2_w4a4_m128 cfg2_w8a8_m128; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"act_quant|gemm_tc" -s 10 -c 6 --csv python bench.py --workload $w --steps 20 --warmup 3 --no-parts --no-cpu --no-check > $O/${T}_${w}_launches.csv 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:gemm_tc -s 5 -c 1 -f -o $O/${T}_gemm_w4a4 python bench.py --workload cfg2_w4a4_m128 --steps 10 --warmup 3 --no-parts --no-cpu --no-check > $O/${T}_ncu.log 2>&1
