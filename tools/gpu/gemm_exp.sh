run() { timeout 300 python bench.py --no-parts --no-cpu --no-check --steps 1000 --warmup 20 "$@" 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,3))"; }
for w in cfg2_w4a4_m128 cfg2_w8a8_m128; do
  for pre in 0 1 2 4; do echo "== $w tc_pre=$pre: $(run --workload $w --tune tc_pre=$pre)"; done
done
for d in 64 128 192; do echo "== trace tc_dbg=$d"; ABQ_TUNE=tc_dbg=$d timeout 300 python tools/trace_gemm.py cfg2_w4a4_m128 f16 2>&1 | grep -v Warn | sed -n 2,7p; done
for pre in 2; do echo "== trace w8a8 tc_pre=$pre"; ABQ_TUNE=tc_pre=$pre timeout 300 python tools/trace_gemm.py cfg2_w8a8_m128 f16 2>&1 | grep -v Warn | sed -n 2,7p; done
