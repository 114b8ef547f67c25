for t in 1 2; do
timeout 1200 python bench.py --workload cfg3_sweep --steps 200 --warmup 10 > gpurun_out/r02_cfg3_sweep.json 2> gpurun_out/r02_cfg3_sweep.err
echo "run $t rc=$?"; grep "cfg3_sweep:" gpurun_out/r02_cfg3_sweep.err | tail -1; grep -i "error" gpurun_out/r02_cfg3_sweep.err | head -3
[ -s gpurun_out/r02_cfg3_sweep.json ] && break
done
