# compute-sanitizer over one invocation of every kernel family; logs -> gpurun_out/
O=gpurun_out; T=${1:-san}
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > $O/${T}_$tool.txt 2>&1
  echo "rc=$?" >> $O/${T}_$tool.txt
done
