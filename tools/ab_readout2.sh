#!/bin/bash
mkdir -p gpurun_out
for v in "" pf1; do
PDSSM_LIB_VARIANT=$v timeout 120 python tools/time_readout.py f32 >> gpurun_out/rd_time.log 2>&1
PDSSM_LIB_VARIANT=$v timeout 120 python tools/time_readout.py bf16 >> gpurun_out/rd_time.log 2>&1
PDSSM_LIB_VARIANT=$v timeout 300 python tools/time_gemm.py >> gpurun_out/rd_time.log 2>&1
done
