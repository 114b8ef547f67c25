./tools/mbicache
for o in f16 f32 f64; do echo "== gemm trace out=$o"; timeout 300 python tools/trace_gemm.py cfg2_w4a4_m128 $o 2>&1 | grep -v Warn | head -12; done
echo "== w8a8"; timeout 300 python tools/trace_gemm.py cfg2_w8a8_m128 f16 2>&1 | grep -v Warn | head -12
