#!/bin/bash
# Subtrees with the warp-wide supernode code: path tests, c2 bench A/B, timeline.
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "level_products" > $O/pytest_paths.log 2>&1
echo "paths rc=$?" >> $O/status.txt
B="python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e"
for kb in 96 48 200; do
QPB_ST_KB=$kb timeout 900 $B > $O/bench_c2_kb$kb.json 2> $O/bench_c2_kb$kb.err
echo "bench c2 kb$kb rc=$?" >> $O/status.txt
done
timeout 600 python scripts/timeline.py c2 12 > $O/timeline_c2.txt 2>&1
QPB_ST=0 timeout 600 python scripts/timeline.py c2 12 > $O/timeline_c2_nost.txt 2>&1
echo "timeline rc=$?" >> $O/status.txt
