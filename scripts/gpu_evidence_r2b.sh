#!/bin/bash
# Round-2 evidence, second pass (after the deterministic reduction and the nested-dissection P_H order).
set -u
O=gpurun_out/ev3
mkdir -p $O
python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/status.txt
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
run c1_W      'k_dense_symv|k_symv_reduce|k_pcg_step' 40 6 python scripts/pcg_once.py c1 40
run c2_root   'k_symroot_gemv|k_symv_reduce'          20 4 python scripts/pcg_once.py c2 25
run c4s_ph_nd 'k_trsv_fwd|k_trsv_bwd'                  40 4 python scripts/pcg_once.py c4s 12 high
# launch list of a short bench run (device times, cold and serialised: shares, not absolutes)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-ipm-solve --secondary "" --no-e2e > $O/launches.log 2>&1
echo "launches rc=$?" >> $O/status.txt
gzip -f $O/launches.csv
du -sh $O
