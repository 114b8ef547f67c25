run() { timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 500 --warmup 20 "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3))"; }
for w in cfg3_w4a8_o_m128 cfg3_w4a8_down_m128 cfg3_w6a6_o_m128 cfg2_w4a4_m128; do
  for tt in 0 64 32; do echo "== $w tc_tt=$tt: $(run --workload $w --tune tc_tt=$tt)"; done
done
