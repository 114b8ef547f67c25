O=gpurun_out; T=${1:-gm}
for w in cfg2_w4a4_m128 cfg2_w8a8_m128; do for tt in 0 64 32; do for s in 0 1 2; do echo "$w tt=$tt sched=$s";
python - <<PY
import sys; sys.argv=['bench.py','--workload','$w','--steps','2000','--warmup','50','--no-cpu','--no-check','--no-parts','--tune','tc_tt=$tt']
import paper_2408_08554_b200 as abq
abq._lib.lib().abq_set_gemm_schedule($s)
import bench; bench.main()
PY
done; done; done > $O/${T}_bench.txt 2>&1
