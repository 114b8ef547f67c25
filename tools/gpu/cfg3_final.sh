for t in 1 2; do
timeout 1200 python bench.py --workload cfg3_sweep --steps 200 --warmup 10 > gpurun_out/r02j_cfg3_sweep.json 2> gpurun_out/r02j_cfg3_sweep.err
[ -s gpurun_out/r02j_cfg3_sweep.json ] && break
done
