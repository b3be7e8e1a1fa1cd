#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/tt_${name}.json 2> gpurun_out/tt_${name}.err; }
for t in 1124 1250 1500 1799 2248; do PDSSM_PATH=seqc run c3_t$t --config 3 --tau $t; done
for t in 2048 2521 3277; do PDSSM_PATH=seqc run c5_t$t --config 5 --tau $t; done
