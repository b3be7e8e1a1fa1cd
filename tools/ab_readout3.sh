#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_project.py tests/test_gpu_select.py tests/test_gpu_surrogate.py tests/test_gpu_block.py tests/test_gpu_scan.py -q -x -k "readout or layer or project or select or block or surrogate or soft" 2>&1 | tail -3 > gpurun_out/rd_pytest.log
timeout 120 python tools/time_readout.py f32 >> gpurun_out/rd_time.log 2>&1
timeout 120 python tools/time_readout.py bf16 >> gpurun_out/rd_time.log 2>&1
timeout 300 python tools/time_gemm.py >> gpurun_out/rd_time.log 2>&1
