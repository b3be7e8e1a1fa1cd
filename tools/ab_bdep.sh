#!/bin/bash
mkdir -p gpurun_out
PDSSM_LIB_VARIANT=bdep timeout 600 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py -q -x 2>&1 | tail -2 > gpurun_out/bd_pytest.log
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/bd_${name}.json 2> gpurun_out/bd_${name}.err; }
for v in "" bdep; do
  PDSSM_LIB_VARIANT=$v run c2_$v
  PDSSM_LIB_VARIANT=$v run c2bf16_$v --dtype bf16
  PDSSM_LIB_VARIANT=$v run c4_$v --config 4
  PDSSM_LIB_VARIANT=$v run c3_$v --config 3
  PDSSM_LIB_VARIANT=$v run c5_$v --config 5
done
