#!/bin/bash
# Round-2 experiment: recompute kernel after the chain fixes, and the GCAP=6 forward variant.
tag=${1:-r02n}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 50 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
timeout 900 python -m pytest tests/test_gpu_recompute.py -q 2>&1 | tail -3
b c2rc --recompute
b c2
PDSSM_LIB_VARIANT=cap6 b c2_cap6
b c2bf16 --dtype bf16
PDSSM_LIB_VARIANT=cap6 b c2bf16_cap6 --dtype bf16
b c4 --config 4
PDSSM_LIB_VARIANT=cap6 b c4_cap6 --config 4
