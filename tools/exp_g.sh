#!/bin/bash
# chunked single-CTA path: tau x group-size sweep (configs 3 and 5)
tag=${1:-r02s}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 30 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
for v in "" seqc16; do
  for t in 1124 1200 1384 1500; do PDSSM_PATH=seqc PDSSM_LIB_VARIANT=$v b c3_g${v:-8}_t$t --config 3 --tau $t; done
  for t in 2341 2521 2731 2979; do PDSSM_LIB_VARIANT=$v b c5_g${v:-8}_t$t --config 5 --tau $t; done
done
