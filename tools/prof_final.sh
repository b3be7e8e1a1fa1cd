#!/bin/bash
# ncu --set full of the scan kernels of every bench config (one fwd + one bwd launch each) and the
# launch list of the default bench command; read here with tools/traffic_json.py / tools/ncu_summary.py
tag=${1:-r02}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled --print-units base --csv --log-file gpurun_out/${tag}_launches_default.csv \
  python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo "launches $?"
for cfg in "c2 --config 2" "c2bf16 --config 2 --dtype bf16" "c3 --config 3" "c4 --config 4" "c5 --config 5"; do
  set -- $cfg; name=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_(fwd|bwd)_(seq|fused)" -s 3 -c 2 -o gpurun_out/${tag}_full_${name} \
    python bench.py --profile --steps 1 --warmup 1 "$@" > /dev/null 2>&1
  echo "$name $?"
done
