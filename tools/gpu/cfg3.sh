timeout 1500 python bench.py --workload cfg3_sweep --steps 200 --warmup 10 > gpurun_out/r02_cfg3_sweep.json 2> gpurun_out/r02_cfg3_sweep.err
timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 2000 --warmup 50 | tail -1 > gpurun_out/head_check.json
