#!/bin/bash
# ncu --set full (source counters) of the single-chunk forward at the bench shape
mkdir -p gpurun_out
TAG=${1:-f1}
ncu --set full --clock-control none --import-source on -k regex:"k_fwd_seq" -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-layer > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep k_fwd_ > gpurun_out/ncu_summary_fwd_${TAG}.txt 2>&1
tail -12 gpurun_out/ncu_summary_fwd_${TAG}.txt
