#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/gf_${name}.json 2> gpurun_out/gf_${name}.err; }
PDSSM_LIB_VARIANT=gf64 run c2bf16_gf64 --dtype bf16
run c2bf16_ --dtype bf16
