mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py -q -x 2>&1 | tail -3 > gpurun_out/pt.log
for dt in f32 bf16; do timeout 300 python bench.py --steps 20 --warmup 5 --dtype $dt --no-cpu-baseline --no-layer --seeds 1 > gpurun_out/b_${dt}.json 2>gpurun_out/b_${dt}.err; done
