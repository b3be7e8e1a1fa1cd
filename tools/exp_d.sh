#!/bin/bash
tag=${1:-r02o}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 50 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
timeout 1200 python -m pytest tests/test_gpu_scan.py tests/test_gpu_recompute.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
b c2
b c2bf16 --dtype bf16
b c4 --config 4
b c5 --config 5
b c2rc --recompute
