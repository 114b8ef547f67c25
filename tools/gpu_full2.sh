O=gpurun_out; T=${1:-full}
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "rc=$?" >> $O/${T}_smoke.log
bash tools/gpu_sanitize.sh $T
