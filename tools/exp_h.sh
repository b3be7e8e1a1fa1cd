#!/bin/bash
tag=${1:-r02t}
b() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-layer --seeds 1 --stat-steps 50 "$@" > gpurun_out/${tag}_${name}.json 2> gpurun_out/${tag}_${name}.err; echo "$name $?"; }
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
b c3 --config 3
b c5 --config 5
b c2
