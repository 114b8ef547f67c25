O=gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > $O/r2_pytest.log 2>&1; echo "rc=$?" >> $O/r2_pytest.log
for w in cfg2_w4a4_m1 cfg1_w2a8 cfg2_w8a8_m1 cfg2_w4a4_m8; do timeout 120 python tools/trace_dec.py $w 8; done > $O/r2_trace.txt 2>&1
for kb in 48 64 80 96; do echo "ring $kb"; ABQ_DEC_RING_KB=$kb timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu --no-check; done > $O/r2_ring.txt 2>&1
ABQ_DEC_PDL=0 timeout 300 python bench.py --steps 5000 --warmup 50 --no-cpu --no-check > $O/r2_nopdl.txt 2>&1
timeout 900 python bench.py --sweep --no-cpu > $O/r2_sweep.json 2> $O/r2_sweep.err
