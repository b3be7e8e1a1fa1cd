#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py -q -x 2>&1 | tail -3 > gpurun_out/sl_pytest.log
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 "$@" > gpurun_out/sl_${name}.json 2> gpurun_out/sl_${name}.err; }
for sl in 1; do
  PDSSM_SEQ_SLOTS=$sl run c2_$sl
  PDSSM_SEQ_SLOTS=$sl run c4_$sl --config 4
  PDSSM_SEQ_SLOTS=$sl run c3_$sl --config 3
done
