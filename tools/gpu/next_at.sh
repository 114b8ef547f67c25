run() { timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 2000 --warmup 50 "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3), d['roofline']['frac'])"; }
for rep in 1 2; do
for at in 100 80 60 40; do echo "== w4a4 next_at=$at: $(run --tune dec_next_at=$at)"; done
echo "== w4a4 next_kb=0: $(run --tune dec_next_kb=0)"
done
