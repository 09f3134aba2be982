#!/bin/bash
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "level_products" > $O/pytest_paths.log 2>&1
echo "paths rc=$?" >> $O/status.txt
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e"
timeout 900 $B --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 $B --config c4s > $O/bench_c4s.json 2> $O/bench_c4s.err
echo "bench rc=$?" >> $O/status.txt
timeout 600 python scripts/timeline.py c2 12 > $O/timeline_c2.txt 2>&1
