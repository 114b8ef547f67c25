run() { timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 2000 --warmup 50 "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3), d['roofline']['frac'])"; }
timeout 900 python -m pytest tests/test_gpu_gemv_variants.py tests/test_gpu_llama_shapes.py tests/test_gpu_ties.py tests/test_gpu_producer.py -x -q 2>&1 | tail -3
for w in cfg2_w4a4_m1 cfg1_w2a8 w2a8_m1_gate_up w2a8_m1_down cfg2_w8a8_m1 cfg2_w4a4_m8; do
  echo "== $w: $(run --workload $w)"
done
timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -12
timeout 300 python tools/trace_dec.py cfg2_w4a4_m1 6 | tail -4
