#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 "$@" > gpurun_out/fv_${name}.json 2> gpurun_out/fv_${name}.err; }
run base
PDSSM_LIB_VARIANT=pred run pred
PDSSM_LIB_VARIANT=gcap6 run gcap6
PDSSM_SEQ_TIER=1 run tier
run base_bf16 --dtype bf16
PDSSM_LIB_VARIANT=gcap6 run gcap6_bf16 --dtype bf16
PDSSM_SEQ_TIER=1 run tier_bf16 --dtype bf16
