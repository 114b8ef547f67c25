O=gpurun_out; T=${1:-tr}
for c in 1 6; do echo "== copies $c"; timeout 120 python tools/trace_dec.py cfg2_w4a4_m1 6 $c 2>&1 | grep -A2 "launch  3"; done > $O/${T}_trace.txt 2>&1
for c in 1 6; do echo "== copies $c"; timeout 120 python tools/trace_dec.py cfg1_w2a8 6 $c 2>&1 | grep -A2 "launch  3"; done >> $O/${T}_trace.txt 2>&1
