#!/bin/bash
# Final check after the three-way F-solve path choice: full GPU suite, smoke, the default bench line, the reference arm,
# c3s / c4s bench lines, the c3s launch list (leaf-phase level products forced) and the c3s timeline.
set -u
O=gpurun_out/fin3
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/status.txt
QPB_VERBOSE=1 timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/status.txt
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e"
for cfg in c3s c4s; do
timeout 900 $B --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
echo "bench small rc=$?" >> $O/status.txt
timeout 900 python scripts/timeline.py c3s 12 > $O/timeline_c3s.txt 2>&1
echo "timeline rc=$?" >> $O/status.txt
export QPB_PROFILE_TIMED=1 QPB_PI=2 QPB_ST=0
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $O/launches_c3s.csv \
    python bench.py --config c3s --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e > $O/launches_c3s.log 2>&1
echo "launches_c3s rc=$?" >> $O/status.txt
gzip -f $O/launches_c3s.csv
