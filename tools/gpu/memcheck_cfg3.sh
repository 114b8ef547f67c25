timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/memcheck_cfg3.log python bench.py --workload cfg3_sweep --steps 4 --warmup 3 --no-cpu > gpurun_out/memcheck_cfg3.out 2>&1
echo "rc=$?"; grep -c "Invalid\|ERROR SUMMARY" gpurun_out/memcheck_cfg3.log; grep "ERROR SUMMARY" gpurun_out/memcheck_cfg3.log; grep -m5 -A12 "Invalid" gpurun_out/memcheck_cfg3.log | head -60
