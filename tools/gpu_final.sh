#!/bin/bash
# End-of-round gpurun session: GPU parity tests, smoke, bench (both arms), ncu launch list + full
# captures of the decode GEMV and the prefill GEMM.  usage (under gpurun): bash tools/gpu_final.sh [tag]
TAG=${1:-r02f}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench20.json 2> $O/${TAG}_bench20.err
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-check --no-parts > $O/${TAG}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_dec -s 20 -c 1 -f -o $O/${TAG}_gemv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-check --no-parts > $O/${TAG}_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 5 -c 1 -f -o $O/${TAG}_gemm \
  python bench.py --workload cfg2_w4a4_m128 --steps 10 --warmup 3 --no-cpu --no-check --no-parts > $O/${TAG}_ncu_gemm.log 2>&1
echo done
timeout 1200 python bench.py --workload cfg3_sweep --steps 200 --warmup 10 > $O/${TAG}_cfg3_sweep.json 2> $O/${TAG}_cfg3_sweep.err
