#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_project.py tests/test_gpu_surrogate.py tests/test_gpu_block.py tests/test_gpu_scan.py -q -x -k "readout or layer or block" 2>&1 | tail -4 > gpurun_out/rd_pytest.log
timeout 120 python tools/time_readout.py f32 >> gpurun_out/rd_time.log 2>&1
PDSSM_READOUT_ATM=0 timeout 120 python tools/time_readout.py f32 >> gpurun_out/rd_time.log 2>&1
timeout 120 python tools/time_readout.py bf16 >> gpurun_out/rd_time.log 2>&1
