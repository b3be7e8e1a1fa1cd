#!/bin/bash
# round-2 experiments: two-tier gather at config 4, 15-warp fused kernels at configs 3/5, readout ncu
tag=${1:-r02x}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_scan.py -q -x -k "paired" 2>&1 | tail -2
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 30 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
b c4_tier --config 4
PDSSM_SEQ_NO_TIER=1 b c4_notier --config 4
b c3 --config 3
PDSSM_LIB_VARIANT=w15 b c3_w15 --config 3
b c5 --config 5
PDSSM_LIB_VARIANT=w15 b c5_w15 --config 5
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiReadout \
  -s 1 -c 1 -o gpurun_out/${tag}_readout python tools/gemm_driver.py > /dev/null 2>&1; echo "ncu readout $?"
