#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sp.py tests/test_gpu_sp_dist.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/sp_pytest.log
timeout 600 python tools/time_sp.py > gpurun_out/sp_time.log 2>&1
