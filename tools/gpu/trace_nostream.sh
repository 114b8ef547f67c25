echo "== W4A4 with stream"; timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -12
echo "== W4A4 no stream"; ABQ_TUNE=dec_dbg_nostream=1 timeout 300 python tools/trace_dec_cta.py cfg2_w4a4_m1 12 | tail -12
echo "== W2A8 q no stream"; ABQ_TUNE=dec_dbg_nostream=1 timeout 300 python tools/trace_dec_cta.py cfg1_w2a8 12 | tail -12
echo "== W4A4 phases no stream"; ABQ_TUNE=dec_dbg_nostream=1 timeout 300 python tools/trace_dec.py cfg2_w4a4_m1 6 | tail -4
