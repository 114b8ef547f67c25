CUDA_LAUNCH_BLOCKING=1 timeout 1200 python bench.py --workload cfg3_sweep --steps 20 --warmup 3 --no-cpu > gpurun_out/cfg3_dbg.json 2> gpurun_out/cfg3_dbg.err
grep "cfg3_sweep:" gpurun_out/cfg3_dbg.err | tail -2
