#!/bin/bash
mkdir -p gpurun_out
PDSSM_LIB_VARIANT=bdb timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2 > gpurun_out/db_pytest.log
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/db_${name}.json 2> gpurun_out/db_${name}.err; }
for v in "" bdb; do
  PDSSM_LIB_VARIANT=$v run c3_$v --config 3
  PDSSM_LIB_VARIANT=$v run c5_$v --config 5
done
