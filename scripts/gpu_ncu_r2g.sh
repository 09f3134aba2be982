#!/bin/bash
# ncu --set full of one PCG iteration's kernels on c4s and c3s with the level products over the leaf phase
# (the path the factor-time timing chooses there; forced, because under ncu every launch is serialised).
set -u
O=gpurun_out/ncu3
mkdir -p $O
export QPB_PI=2 QPB_ST=0
for cfg in c4s c3s; do
  timeout 600 python scripts/pcg_once.py $cfg 12 > $O/${cfg}_plain.log 2>&1 || { echo "$cfg plain failed" >> $O/status.txt; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on \
     -k "regex:k_pi_|k_lvl16_|k_pcg_step|k_symroot_gemv|k_symv_reduce" -s 120 -c 45 -o $O/${cfg}_iter \
     python scripts/pcg_once.py $cfg 12 > $O/${cfg}_ncu.log 2>&1
  echo "$cfg ncu rc=$?" >> $O/status.txt
  if [ -f $O/${cfg}_iter.ncu-rep ]; then
    ncu -i $O/${cfg}_iter.ncu-rep --page raw --csv > $O/${cfg}_iter.raw.csv 2>/dev/null
    rm -f $O/${cfg}_iter.ncu-rep
  fi
done
