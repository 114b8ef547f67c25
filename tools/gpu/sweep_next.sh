set -x
for w in cfg2_w4a4_m1 cfg1_w2a8 w2a8_m1_gate_up w2a8_m1_down cfg2_w8a8_m1; do
  for kb in 0 32 64 128; do
    echo "== $w next_kb=$kb"
    timeout 300 python bench.py --workload $w --no-parts --no-cpu --no-check --steps 2000 --warmup 50 --tune dec_next_kb=$kb 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']*1e3, d['roofline']['frac'], d['e2e']['ms_per_step']*1e3)"
  done
done
timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12
