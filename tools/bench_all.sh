#!/bin/bash
# Every §8(d) bench line on one GPU (run under gpurun): the default headline line, then the
# other configs / dtypes / the recompute backward.  Output: gpurun_out/<tag>_bench_*.json
tag=${1:-r02}
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/${tag}_bench_${name}.json 2> gpurun_out/${tag}_bench_${name}.err; echo "$name rc=$?"; }
run c2 --steps 20 --warmup 5
run c2bf16 --dtype bf16 --no-layer --no-cpu-baseline --seeds 1
run c2rc --recompute --no-layer --no-cpu-baseline --seeds 1
run c4 --config 4 --no-cpu-baseline
run c3 --config 3 --no-cpu-baseline
run c5 --config 5 --no-cpu-baseline
run ref2 --impl reference --config 2
