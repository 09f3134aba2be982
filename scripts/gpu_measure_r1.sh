set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^k_(?!flat_extract|set_unit)' --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ipm-solve > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_flat_fwd_t|k_flat_bwd_t|k_symroot_gemv|k_pcg_step' -s 40 -c 4 -o gpurun_out/r1_full python scripts/pcg_once.py c1 40 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/ncu_full.log
