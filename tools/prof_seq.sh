#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-s1}
PATHS=seq ncu --set full --clock-control none --import-source on -k regex:"k_(fwd|bwd)_seq" -s 2 -c 2 -o gpurun_out/prof_${TAG} python tools/diag_paths.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep k_fwd_seq > gpurun_out/sum_${TAG}_fwd.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep k_bwd_seq > gpurun_out/sum_${TAG}_bwd.txt 2>&1
ls -la gpurun_out/prof_${TAG}.ncu-rep
