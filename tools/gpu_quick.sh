# quick GPU iteration: decode-GEMV parity tests, phase trace, bench lines
O=gpurun_out; T=${1:-q}
timeout 600 python -m pytest tests/test_gpu_gemv_variants.py tests/test_gpu_parity.py -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for w in cfg2_w4a4_m1 cfg1_w2a8 cfg2_w8a8_m1; do timeout 120 python tools/trace_dec.py $w 6; done > $O/${T}_trace.txt 2>&1
timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu --no-check > $O/${T}_bench.json 2>&1
timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu --no-check --no-prefetch-next > $O/${T}_bench_nonext.json 2>&1
for w in cfg1_w2a8 cfg2_w8a8_m1 cfg2_w4a4_m8; do timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu --no-check --workload $w; done > $O/${T}_bench_more.json 2>&1
