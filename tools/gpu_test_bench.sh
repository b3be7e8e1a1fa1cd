#!/bin/bash
# usage: bash tools/gpu_test_bench.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$K" 2>&1 | tail -40 > gpurun_out/pytest.log
else
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -40 > gpurun_out/pytest.log
fi
cat gpurun_out/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -3 | tee gpurun_out/bench.log
