O=gpurun_out; T=${1:-prod}
timeout 900 python -m pytest tests/test_gpu_producer.py tests/test_gpu_gemv_variants.py -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
for w in llama7b_decode_chain_w4a4 llama7b_decode_chain_w2a8; do
  for kb in -1 64 1024; do echo "$w pre_kb=$kb"; timeout 300 python bench.py --workload $w --steps 500 --warmup 20 --tune dec_pre_kb=$kb; done
done > $O/${T}_chain.txt 2>&1
