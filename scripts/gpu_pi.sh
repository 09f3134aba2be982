#!/bin/bash
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
for i in 1 2 3; do
timeout 1500 python -m pytest tests/test_gpu_full.py tests/test_gpu_consistent.py tests/test_gpu_sharded_mp.py tests/test_gpu_sharded.py -m gpu -q > $O/pytest_$i.log 2>&1
echo "pytest $i rc=$?" >> $O/status.txt
done
timeout 900 python scripts/c2_counts.py c2 6 5 > $O/counts_c2.txt 2>&1
timeout 900 python scripts/c2_counts.py c4s 4 6 > $O/counts_c4s.txt 2>&1
