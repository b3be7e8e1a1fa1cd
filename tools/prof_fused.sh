#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-v2}
ncu --set full --clock-control none --import-source on -k regex:k_bwd_fused -s 1 -c 1 -o gpurun_out/prof_${TAG}_bwd python tools/diag_paths.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fwd_fused -s 1 -c 1 -o gpurun_out/prof_${TAG}_fwd python tools/diag_paths.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -2
