run() { timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 2000 --warmup 50 "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3), d['roofline']['frac'])"; }
for w in cfg2_w4a4_m1 w2a8_m1_gate_up; do
  for pl in 0 1; do
    for kb in 0 64 256; do
      echo "== $w l2_plain=$pl next_kb=$kb min=0: $(run --workload $w --tune dec_l2_plain=$pl --tune dec_next_kb=$kb --tune dec_next_min_kb=0)"
    done
  done
done
echo "== cfg1_w2a8 default: $(run --workload cfg1_w2a8)"
echo "== cfg2_w4a4_m1 default: $(run --workload cfg2_w4a4_m1)"
ABQ_NEXT=0 timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -12
ABQ_NEXT=1 timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -12
