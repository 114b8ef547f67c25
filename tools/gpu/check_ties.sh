run() { timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 2000 --warmup 50 "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3), d['roofline']['frac'])"; }
timeout 600 python -m pytest tests/test_gpu_ties.py tests/test_cpp_api.py -x -q 2>&1 | tail -5
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -5
for w in cfg2_w4a4_m1 cfg1_w2a8 w2a8_m1_gate_up w2a8_m1_down cfg2_w8a8_m1 cfg2_w8a8_m128 cfg2_w4a4_m128; do
  echo "== $w: $(run --workload $w)"
done
timeout 300 python tools/trace_dec_cta.py cfg1_w2a8 12 | tail -10
timeout 300 python tools/trace_dec.py cfg1_w2a8 6 | tail -6
