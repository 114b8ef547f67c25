O=gpurun_out; T=${1:-dec}
timeout 900 python -m pytest tests/test_gpu_gemv_variants.py tests/test_gpu_producer.py tests/test_gpu_llama_shapes.py tests/test_gpu_parity.py -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for w in cfg2_w4a4_m1 cfg1_w2a8; do timeout 120 python tools/trace_dec.py $w 6; done > $O/${T}_trace.txt 2>&1
for w in cfg2_w4a4_m1 w2a8_m1_gate_up cfg1_w2a8 w2a8_m1_down cfg2_w8a8_m1 cfg2_w4a4_m8 llama7b_decode_chain_w4a4; do
  echo "$w"; timeout 300 python bench.py --workload $w --steps 2000 --warmup 50 --no-cpu --no-check --no-parts
done > $O/${T}_bench.txt 2>&1
