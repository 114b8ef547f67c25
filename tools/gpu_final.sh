#!/bin/bash
# Short end-of-round gpurun session: GPU parity tests, smoke, bench (both arms), ncu launch list + full
# capture of the decode GEMV.  usage (under gpurun): bash tools/gpu_final.sh [tag]
TAG=${1:-r01f}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-check > $O/${TAG}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_dec -s 20 -c 3 -f -o $O/${TAG}_gemv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-check > $O/${TAG}_ncu_full.log 2>&1
echo done
