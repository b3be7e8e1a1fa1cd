#!/bin/bash
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 "$@" > gpurun_out/sq_${name}.json 2> gpurun_out/sq_${name}.err; }
for tau in 256 512 1024; do
  PDSSM_PATH=seqc run bf16_t$tau --dtype bf16 --tau $tau
  PDSSM_PATH=seqc run f32_t$tau --tau $tau
done
PDSSM_PATH=seqc run c4_t1024 --config 4 --tau 1024
PDSSM_PATH=seqc run c4_t2048 --config 4 --tau 2048
