#!/bin/bash
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_operator.py tests/test_gpu_sharded.py tests/test_gpu_sharded_mp.py tests/test_gpu_xspace.py -m gpu -q > $O/pytest_op.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 1500 python scripts/operator_full.py c3 20 > $O/operator_c3.json 2> $O/operator_c3.err
echo "op c3 rc=$?" >> $O/status.txt
timeout 2400 python scripts/operator_full.py c4 20 > $O/operator_c4.json 2> $O/operator_c4.err
echo "op c4 rc=$?" >> $O/status.txt
