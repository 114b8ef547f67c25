O=gpurun_out; T=${1:-gm}
timeout 900 python -m pytest tests/test_gpu_gemm_tc.py tests/test_gpu_llama_shapes.py tests/test_gpu_parity.py -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for w in cfg2_w4a4_m128 cfg2_w8a8_m128 cfg2_w4a4_m16; do echo $w; timeout 300 python bench.py --workload $w --steps 2000 --warmup 50 --no-cpu --no-check --no-parts; done > $O/${T}_bench.txt 2>&1
for w in cfg2_w4a4_m128; do timeout 120 python tools/trace_gemm.py $w f16 classic 2>&1 | head -8; done > $O/${T}_trace.txt 2>&1
