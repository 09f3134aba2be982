#!/bin/bash
# Round-2 evidence pass (one gpurun call): fp64 peak, then ncu --set full captures of the kernels the
# verdict asked for, each preceded by the same command run plainly (B200_PROFILING.md).
set -u
O=gpurun_out/ev2
mkdir -p $O
python scripts/fp64_peak.py > $O/fp64_peak.json 2> $O/fp64_peak.err
run() {   # name, kernel regex, skip, count, command...
  local name=$1 rx=$2 sk=$3 ct=$4; shift 4
  "$@" > $O/$name.plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $sk -c $ct -o $O/$name "$@" > $O/$name.ncu.log 2>&1
  echo "$name rc=$?" >> $O/status.txt
  # bring back text only (gpurun returns at most 64 MiB): the raw metrics and the details page
  if [ -f $O/$name.ncu-rep ]; then
    ncu -i $O/$name.ncu-rep --page raw --csv > $O/$name.raw.csv 2>/dev/null
    ncu -i $O/$name.ncu-rep --page details --csv > $O/$name.details.csv 2>/dev/null
    rm -f $O/$name.ncu-rep
  fi
}
run c1_W      'k_dense_symv|k_pcg_step'            40 4 python scripts/pcg_once.py c1 40
run c2_sweeps 'k_trsv_fwd|k_trsv_bwd|k_symroot_gemv' 30 3 python scripts/pcg_once.py c2 25
run c4s_ph    'k_trsv_fwd|k_trsv_bwd'               40 4 python scripts/pcg_once.py c4s 12 high
run c4s_sweeps 'k_trsv_fwd|k_trsv_bwd'              20 2 python scripts/pcg_once.py c4s 15
run c3s_sweeps 'k_trsv_fwd|k_trsv_bwd'              20 2 python scripts/pcg_once.py c3s 15
run ipm_a9    'k_ipm'                                 0 6 python scripts/pcg_once.py c3s 2 low ipm
