#!/bin/bash
# ncu launch lists (device time per launch; cold-cache, serialised) for every bench config.
tag=${1:-r02}
mkdir -p gpurun_out
for cfg in "c2 --config 2" "c2bf16 --config 2 --dtype bf16" "c2rc --config 2 --recompute" "c3 --config 3" "c4 --config 4" "c5 --config 5"; do
  set -- $cfg; name=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled --print-units base \
    -k regex:pdssm --csv --log-file gpurun_out/${tag}_launches_${name}.csv \
    python bench.py --profile --steps 2 --warmup 1 "$@" > /dev/null 2> gpurun_out/${tag}_launches_${name}.err
  echo "$name rc=$?"
done
