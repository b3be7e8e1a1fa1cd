#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_surrogate.py tests/test_gpu_block.py -q -x -k "layer" 2>&1 | tail -3 > gpurun_out/ly_pytest.log
for a in 1 0; do
  PDSSM_LAYER_ATM=$a timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --seeds 1 --no-e2e > gpurun_out/ly_$a.json 2> gpurun_out/ly_$a.err
done
