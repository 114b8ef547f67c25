# GPU round check: full -m gpu suite, the driver-shaped bench, a longer bench
O=gpurun_out; T=${1:-chk}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo "rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench20.json 2> $O/${T}_bench20.err
timeout 600 python bench.py --steps 2000 --warmup 50 --no-cpu > $O/${T}_bench2000.json 2> $O/${T}_bench2000.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref.json 2>&1
