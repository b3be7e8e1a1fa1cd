#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py tests/test_gpu_sp.py -q -x 2>&1 | tail -2 > gpurun_out/sk_pytest.log
run() { name=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-layer --seeds 1 --no-e2e "$@" > gpurun_out/sk_${name}.json 2> gpurun_out/sk_${name}.err; }
for v in "" noskew; do
  PDSSM_LIB_VARIANT=$v run c3_$v --config 3
  PDSSM_LIB_VARIANT=$v run c5_$v --config 5
  PDSSM_LIB_VARIANT=$v run c4_$v --config 4
done
run c2
