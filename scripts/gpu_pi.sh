#!/bin/bash
# Batched fused step: parity (paths, full c2/c4s), c2 bench on/off, timeline, c4s.
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_paths.py -m gpu -x -q > $O/pytest_paths.log 2>&1
echo "paths rc=$?" >> $O/status.txt
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e"
timeout 900 $B --config c2 > $O/bench_c2.json 2> $O/bench_c2.err
echo "bench c2 rc=$?" >> $O/status.txt
QPB_STEP_B4=0 timeout 900 $B --config c2 > $O/bench_c2_nob4.json 2> $O/bench_c2_nob4.err
timeout 600 python scripts/timeline.py c2 12 > $O/timeline_c2.txt 2>&1
for cfg in c4s c3s; do
timeout 900 $B --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
echo "bench c4s c3s rc=$?" >> $O/status.txt
timeout 2400 python -m pytest tests/test_gpu_full.py -m gpu -x -q --deselect "tests/test_gpu_full.py::test_full_ph_ipm_objective[c1]" > $O/pytest_full.log 2>&1
echo "full rc=$?" >> $O/status.txt
