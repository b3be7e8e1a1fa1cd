#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/rc_${name}.json 2> gpurun_out/rc_${name}.err; }
for tau in 64 96 128 192; do run t$tau --recompute --tau $tau; done
run bf16_t64 --recompute --tau 64 --dtype bf16
run bf16_t192 --recompute --tau 192 --dtype bf16
