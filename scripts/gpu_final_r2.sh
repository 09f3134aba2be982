#!/bin/bash
# Round-2 final check: full GPU suite, smoke, the default bench line (c1 + c2 secondary), and the launch list
# of the c2 bench's timed steps with the level products forced (under ncu the factor-time timing would
# otherwise pick the task graph: every launch is serialised there).
set -u
O=gpurun_out/final${1:-}
mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/status.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/status.txt
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/status.txt
export QPB_PROFILE_TIMED=1 QPB_PI=2
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e > $O/bench_short_c2.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e > $O/launches_c2.log 2>&1
echo "launches_c2 rc=$?" >> $O/status.txt
unset QPB_PROFILE_TIMED QPB_PI
gzip -f $O/launches_c2.csv
QPB_PI=2 bash -c 'python scripts/pcg_once.py c2 12 > '$O'/c2_iter.plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:k_pi_|k_st16_|k_pcg_step|k_symroot_gemv|k_symv_reduce" -s 80 -c 40 -o '$O'/c2_iter python scripts/pcg_once.py c2 12 > '$O'/c2_iter.ncu.log 2>&1'
echo "ncu c2 rc=$?" >> $O/status.txt
if [ -f $O/c2_iter.ncu-rep ]; then
  ncu -i $O/c2_iter.ncu-rep --page raw --csv > $O/c2_iter.raw.csv 2>/dev/null
  rm -f $O/c2_iter.ncu-rep
fi
timeout 900 python scripts/timeline.py c2 12 > $O/timeline_c2.txt 2>&1
timeout 900 python scripts/timeline.py c4s 12 > $O/timeline_c4s.txt 2>&1
echo "timeline rc=$?" >> $O/status.txt
