# Round-1 refresh (run under gpurun): device timelines of the PL PCG on every config, full IPM solves.
for c in c1 c2 c3s c4s; do timeout 600 python scripts/timeline.py $c 40 > gpurun_out/tlr_$c.log 2>&1; done
for cp in "c0 low" "c1 high" "c4s high" "c3s high" "c1 low"; do
  set -- $cp
  timeout 900 python scripts/ipm_probe.py $1 $2 2000 > gpurun_out/ipm_$1_$2.log 2>&1
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
