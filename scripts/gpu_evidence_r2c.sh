#!/bin/bash
# Round-2 evidence, third pass: the PCG's W product, the launch list of the bench's timed steps, and the
# consistent-protocol PL-KF runs on c1, c4s and c3s.
set -u
O=gpurun_out/ev4
mkdir -p $O
run() {
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  "$@" > $O/$name.plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $sk -c $ct -o $O/$name "$@" > $O/$name.ncu.log 2>&1
  echo "$name rc=$?" >> $O/status.txt
  if [ -f $O/$name.ncu-rep ]; then
    ncu -i $O/$name.ncu-rep --page raw --csv > $O/$name.raw.csv 2>/dev/null
    ncu -i $O/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
    rm -f $O/$name.ncu-rep
  fi
}
run c1_W 'k_dense_symv|k_pcg_step' 2 4 python scripts/pcg_once.py c1 40
export QPB_PROFILE_TIMED=1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_short.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/launches.log 2>&1
echo "launches rc=$?" >> $O/status.txt
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_short_c2.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/launches_c2.log 2>&1
echo "launches_c2 rc=$?" >> $O/status.txt
unset QPB_PROFILE_TIMED
gzip -f $O/launches.csv $O/launches_c2.csv
for c in c1 c4s c3s; do timeout 900 python scripts/consistent_pl.py $c 2000 > $O/consistent_$c.json 2> $O/consistent_$c.err; done
echo "consistent rc=$?" >> $O/status.txt
du -sh $O
