#!/bin/bash
# Programmatic dependent launch in the level-product chain: path tests, c2 bench on/off, timeline, c4s.
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "level_products" > $O/pytest_paths.log 2>&1
echo "paths rc=$?" >> $O/status.txt
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e"
QPB_VERBOSE=1 timeout 900 $B --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
echo "bench c2 rc=$?" >> $O/status.txt
QPB_PDL=0 timeout 900 $B --config c2 > $O/bench_c2_nopdl.json 2> $O/bench_c2_nopdl.err
QPB_NO_GRAPH=1 timeout 900 $B --config c2 > $O/bench_c2_nograph.json 2> $O/bench_c2_nograph.err
timeout 600 python scripts/timeline.py c2 12 > $O/timeline_c2.txt 2>&1
for cfg in c4s c3s; do
QPB_VERBOSE=1 timeout 900 $B --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
echo "bench c4s c3s rc=$?" >> $O/status.txt
