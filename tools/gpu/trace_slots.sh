ABQ_NEXT=0 timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -24
ABQ_NEXT=1 timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -13
timeout 300 python tools/trace_dec_cta.py cfg1_w2a8 12 | tail -13
