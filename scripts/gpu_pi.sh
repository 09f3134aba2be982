#!/bin/bash
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/status.txt
