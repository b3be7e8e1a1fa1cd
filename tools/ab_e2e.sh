#!/bin/bash
mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-layer --seeds 1 > gpurun_out/e2e_c2.json 2> gpurun_out/e2e_c2.err
timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-layer --seeds 1 > gpurun_out/e2e_c4.json 2> gpurun_out/e2e_c4.err
timeout 600 python -m pytest tests/test_gpu_bench_multirank.py -q -x 2>&1 | tail -3 > gpurun_out/e2e_pytest.log
