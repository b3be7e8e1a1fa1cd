#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/pm_${name}.json 2> gpurun_out/pm_${name}.err; }
for c in 4 5 6 7; do PDSSM_SEQ_MAX_PER_SM=$c run c4_$c --config 4; done
for c in 2 3 4; do PDSSM_SEQ_MAX_PER_SM=$c run c3_$c --config 3; done
