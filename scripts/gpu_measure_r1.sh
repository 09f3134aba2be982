# Round-1 measurement batch (run under gpurun): bench line, ncu launch list of the bench command,
# ncu --set full of the dominant kernels of a c1 PCG solve.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^k_(?!flat_extract|set_unit)' --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ipm-solve > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/ncu_launch.log
