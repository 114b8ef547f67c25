O=gpurun_out; T=${1:-dec}
timeout 900 python -m pytest tests/test_gpu_gemv_variants.py tests/test_gpu_producer.py tests/test_gpu_llama_shapes.py tests/test_gpu_parity.py -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for w in cfg2_w4a4_m1 cfg1_w2a8; do timeout 120 python tools/trace_dec.py $w 6; done > $O/${T}_trace.txt 2>&1
for w in cfg2_w4a4_m1 w2a8_m1_gate_up cfg1_w2a8 w2a8_m1_down cfg2_w8a8_m1 cfg2_w4a4_m8; do
  for p in 0 25 50; do echo "$w pace=$p"; timeout 300 python bench.py --workload $w --steps 2000 --warmup 50 --no-cpu --no-check --no-parts --tune dec_pace_ns=$p; done
done > $O/${T}_bench.txt 2>&1
echo llama7b_decode_chain_w4a4 >> $O/${T}_bench.txt; timeout 300 python bench.py --workload llama7b_decode_chain_w4a4 --steps 500 --warmup 20 >> $O/${T}_bench.txt 2>&1
