#!/bin/bash
# Leaf-phase (level kernels) check: GPU suite with the default threshold and with every eligible level forced,
# then the c2 sweep trace and a short c2 bench.
set -u
O=gpurun_out/lvl${1:-}
mkdir -p $O
DS="--deselect tests/test_gpu_full.py::test_full_ph_ipm_objective[c1]"
timeout 1500 python -m pytest tests -m gpu -x -q $DS > $O/pytest_default.log 2>&1
echo "pytest default rc=$?" >> $O/status.txt
QPB_LVL_MIN=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_paths.py -m gpu -x -q $DS > $O/pytest_forced.log 2>&1
echo "pytest forced rc=$?" >> $O/status.txt
timeout 600 python scripts/sweep_trace.py c2 > $O/trace_c2.txt 2>&1
echo "trace rc=$?" >> $O/status.txt
timeout 900 python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
echo "bench c2 rc=$?" >> $O/status.txt
QPB_LVL=0 timeout 900 python bench.py --config c2 --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_c2_off.json 2> $O/bench_c2_off.err
echo "bench c2 off rc=$?" >> $O/status.txt
