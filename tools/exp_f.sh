#!/bin/bash
# chunked single-CTA path with small groups (2+ CTAs per SM): config 3 / 5 over tau
tag=${1:-r02r}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 30 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
timeout 1200 python -m pytest tests/test_gpu_scan.py tests/test_gpu_paths.py tests/test_gpu_fullsize.py -q -x -k "seqc or fullsize or config3" 2>&1 | tail -2
b c3 --config 3
PDSSM_PATH=seqc b c3_seqc_t1999 --config 3 --tau 1999
PDSSM_PATH=seqc b c3_seqc_t1799 --config 3 --tau 1799
PDSSM_PATH=seqc b c3_seqc_t1384 --config 3 --tau 1384
PDSSM_PATH=seqc b c3_seqc_t1000 --config 3 --tau 1000
PDSSM_PATH=seqc PDSSM_LIB_VARIANT=seqc16 b c3_seqc16_t1999 --config 3 --tau 1999
b c5 --config 5
PDSSM_LIB_VARIANT=seqc16 b c5_seqc16 --config 5
b c5_t2731 --config 5 --tau 2731
b c5_t4096 --config 5 --tau 4096
