#!/bin/bash
set -u
O=gpurun_out/pi${1:-}
mkdir -p $O
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 scripts/dbg_worker.py > $O/dbg.log 2>&1
echo "dbg rc=$?" >> $O/status.txt
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e"
for cfg in c2 c4s; do
QPB_PI_PF=2 timeout 900 $B --config $cfg > $O/bench_${cfg}_pf2.json 2> $O/bench_${cfg}_pf2.err
timeout 900 $B --config $cfg > $O/bench_${cfg}.json 2> $O/bench_${cfg}.err
done
echo "bench rc=$?" >> $O/status.txt
timeout 600 python scripts/c2_counts.py c3s 4 3 > $O/counts_c3s.txt 2>&1
