#!/bin/bash
# Level products check: path test, full-size parity (c2/c3s/c4s), c2 bench with and without.
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "level_products" > $O/pytest_paths.log 2>&1
echo "paths rc=$?" >> $O/status.txt
QPB_VERBOSE=1 timeout 900 python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
echo "bench c2 rc=$?" >> $O/status.txt
QPB_PI=0 timeout 900 python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_c2_off.json 2> $O/bench_c2_off.err
echo "bench c2 off rc=$?" >> $O/status.txt
timeout 2400 python -m pytest tests/test_gpu_full.py tests/test_gpu_scale.py -m gpu -x -q --deselect "tests/test_gpu_full.py::test_full_ph_ipm_objective" > $O/pytest_full.log 2>&1
echo "full rc=$?" >> $O/status.txt
timeout 600 python scripts/timeline.py c2 > $O/timeline_c2.txt 2>&1
echo "timeline rc=$?" >> $O/status.txt
