# ncu source-level capture of the decode GEMV (headline W4A4 and W2A8 gate/up) + phase traces
O=gpurun_out; T=${1:-pd}
mkdir -p $O
for w in cfg2_w4a4_m1 w2a8_m1_gate_up; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_dec -s 20 -c 1 -f -o $O/${T}_$w \
    python bench.py --workload $w --steps 30 --warmup 3 --no-parts --no-cpu --no-check > $O/${T}_${w}_ncu.log 2>&1
done
for w in cfg2_w4a4_m1 cfg1_w2a8 w2a8_m1_gate_up w2a8_m1_down; do timeout 120 python tools/trace_dec.py $w 6; done > $O/${T}_trace.txt 2>&1
