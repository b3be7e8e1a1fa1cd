#!/bin/bash
# predicated gather slots vs the zero-slot reads (variant nopred)
tag=${1:-r02q}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 50 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
timeout 1200 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py -q -x 2>&1 | tail -2
b c2
PDSSM_LIB_VARIANT=nopred b c2_nopred
b c2bf16 --dtype bf16
PDSSM_LIB_VARIANT=nopred b c2bf16_nopred --dtype bf16
b c4 --config 4
PDSSM_LIB_VARIANT=nopred b c4_nopred --config 4
b c5 --config 5
PDSSM_LIB_VARIANT=nopred b c5_nopred --config 5
