#!/bin/bash
# ncu --set full capture of the tcgen05 GEMMs (tensor-pipe evidence); read here with
# python tools/ncu_summary.py / ncu -i ... --page raw --csv
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_gemm_tc \
  -s 6 -c 6 -o gpurun_out/${tag}_gemm python tools/gemm_driver.py > gpurun_out/${tag}_gemm.log 2>&1
echo "gemm rc=$?"
