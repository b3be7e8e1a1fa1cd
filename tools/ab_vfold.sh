#!/bin/bash
mkdir -p gpurun_out
PDSSM_LIB_VARIANT=vfold timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/vf_pytest.log
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/vf_${name}.json 2> gpurun_out/vf_${name}.err; }
for v in "" vfold; do
  PDSSM_LIB_VARIANT=$v run c2_$v
  PDSSM_LIB_VARIANT=$v run c2bf16_$v --dtype bf16
done
