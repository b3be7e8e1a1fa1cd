#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/pb_${name}.json 2> gpurun_out/pb_${name}.err; }
run c4 --config 4
PDSSM_SEQ_PAIR_BWD=1 run c4_pair --config 4
