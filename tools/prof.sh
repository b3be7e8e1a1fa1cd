set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_v1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench_v1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fwd_phase -s 4 -c 3 -o gpurun_out/prof_v1_fwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_phase -s 4 -c 3 -o gpurun_out/prof_v1_bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
