O=gpurun_out; T=${1:-tr}
for w in cfg1_w2a8 cfg2_w4a4_m1 w2a8_m1_gate_up; do timeout 120 python tools/trace_dec.py $w 6; done > $O/${T}_trace.txt 2>&1
