#!/bin/bash
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
timeout 1500 python scripts/operator_full.py c3 20 > $O/operator_c3.json 2> $O/operator_c3.err
echo "op c3 rc=$?" >> $O/status.txt
timeout 2400 python scripts/operator_full.py c4 20 > $O/operator_c4.json 2> $O/operator_c4.err
echo "op c4 rc=$?" >> $O/status.txt
timeout 3000 python scripts/operator_halo_full.py c4 2 > $O/operator_halo_c4.json 2> $O/operator_halo_c4.err
echo "halo c4 rc=$?" >> $O/status.txt
