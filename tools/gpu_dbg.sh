O=gpurun_out; T=${1:-dbg}
timeout 900 python -m pytest tests/test_gpu_gemm_tc.py -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for d in 0 64; do echo "== ABQ_TC_DBG=$d"; ABQ_TC_DBG=$d timeout 120 python tools/trace_gemm.py cfg2_w4a4_m128 2>&1 | head -28; done > $O/${T}_trace.txt 2>&1
echo "== W8" >> $O/${T}_trace.txt; timeout 120 python tools/trace_gemm.py cfg2_w8a8_m128 2>&1 | head -28 >> $O/${T}_trace.txt
echo "== SK=1" >> $O/${T}_trace.txt; ABQ_TC_SK=1 timeout 120 python tools/trace_gemm.py cfg2_w4a4_m128 2>&1 | head -14 >> $O/${T}_trace.txt
for w in cfg2_w4a4_m128 cfg2_w8a8_m128 cfg2_w4a4_m16; do timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu --no-check --workload $w; ABQ_TC_SK=1 timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu --no-check --workload $w; done > $O/${T}_bench.json 2>&1
