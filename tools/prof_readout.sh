#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_gemm_tc" -s 3 -c 1 \
  -o gpurun_out/rd_full python tools/time_readout.py f32 > /dev/null 2>&1
echo "ncu $?"
python tools/ncu_summary.py gpurun_out/rd_full.ncu-rep k_gemm_tc > gpurun_out/rd_summary.txt 2>&1
ncu -i gpurun_out/rd_full.ncu-rep --page raw --csv > gpurun_out/rd_raw.csv 2>/dev/null
