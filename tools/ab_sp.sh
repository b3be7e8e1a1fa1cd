#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sp.py tests/test_gpu_sp_dist.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -15 > gpurun_out/sp_pytest.log
