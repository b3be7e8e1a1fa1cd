#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/ct_${name}.json 2> gpurun_out/ct_${name}.err; }
run c4_tier --config 4
PDSSM_SEQ_NO_TIER=1 run c4_notier_early --config 4
run c2 
