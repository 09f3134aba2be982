#!/bin/bash
# Round-2 re-entry check: full GPU suite, bench line, c2 sweep trace.
set -u
O=gpurun_out/r2d
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/status.txt
timeout 600 python scripts/sweep_trace.py c2 > $O/trace_c2.txt 2>&1
echo "trace rc=$?" >> $O/status.txt
