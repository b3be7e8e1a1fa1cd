#!/bin/bash
tag=${1:-r02y}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 50 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
b c2
PDSSM_SEQ_TIER=1 b c2_tier
b c2bf16 --dtype bf16
PDSSM_SEQ_TIER=1 b c2bf16_tier --dtype bf16
b c2_t64 --tau 64
b c2bf16_t64 --dtype bf16 --tau 64
b c4 --config 4
