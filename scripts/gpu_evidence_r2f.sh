#!/bin/bash
# Round-2 evidence, level products: ncu --set full of one c2 PCG iteration's kernels (after the plain run
# exits 0), and the launch list of the c2 bench's timed steps.
set -u
O=gpurun_out/ev5
mkdir -p $O
run() {
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  "$@" > $O/$name.plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $sk -c $ct -o $O/$name "$@" > $O/$name.ncu.log 2>&1
  echo "$name rc=$?" >> $O/status.txt
  if [ -f $O/$name.ncu-rep ]; then
    ncu -i $O/$name.ncu-rep --page raw --csv > $O/$name.raw.csv 2>/dev/null
    ncu -i $O/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
    ncu -i $O/$name.ncu-rep --page source --csv -k k_pcg_step > $O/$name.source_pcg_step.csv 2>/dev/null
    rm -f $O/$name.ncu-rep
  fi
}
run c2_iter 'k_pi_|k_st16_|k_pcg_step|k_symroot_gemv|k_symv_reduce' 80 40 python scripts/pcg_once.py c2 12
export QPB_PROFILE_TIMED=1
python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e > $O/bench_short_c2.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary= --no-e2e > $O/launches_c2.log 2>&1
echo "launches_c2 rc=$?" >> $O/status.txt
unset QPB_PROFILE_TIMED
gzip -f $O/launches_c2.csv
du -sh $O
