O=gpurun_out; T=${1:-ncd}
for w in cfg1_w2a8 cfg2_w4a4_m1; do
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:gemv_dec -s 20 -c 1 -f -o $O/${T}_$w \
    python bench.py --workload $w --steps 30 --warmup 3 --no-parts --no-cpu --no-check --tune dec_pre_kb=0 > $O/${T}_${w}_ncu.log 2>&1
done
