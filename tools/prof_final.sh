#!/bin/bash
# ncu --set full of the scan kernels of every bench config (one fwd + one bwd launch each) and the
# launch list of the default bench command.  The reports are summarised ON THE BOX (gpurun brings
# back <= 64 MiB): per-config ncu summaries, DRAM traffic per launch (profiles/traffic_latest.json
# format) and the source-level stall table of the config-2 forward; only the c2 report is kept.
tag=${1:-r02}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled --print-units base --csv --log-file gpurun_out/${tag}_launches_default.csv \
  python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1; echo "launches $?"
rm -f gpurun_out/${tag}_traffic.json
for cfg in "c2 config2 --config 2" "c2bf16 config2_bf16 --config 2 --dtype bf16" "c3 config3 --config 3" "c4 config4 --config 4" "c5 config5 --config 5"; do
  set -- $cfg; name=$1; key=$2; shift 2
  rep=gpurun_out/${tag}_full_${name}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_(fwd|bwd)_(seq|fused)" -s 3 -c 2 -o $rep python bench.py --profile --steps 1 --warmup 1 "$@" > /dev/null 2>&1
  echo "$name $?"
  python tools/ncu_summary.py $rep.ncu-rep "_fwd_" > gpurun_out/${tag}_ncu_summary_${name}_fwd.txt 2>&1
  python tools/ncu_summary.py $rep.ncu-rep "_bwd_" > gpurun_out/${tag}_ncu_summary_${name}_bwd.txt 2>&1
  python tools/traffic_json.py $rep.ncu-rep gpurun_out/${tag}_traffic.json "$key:" > /dev/null 2>&1
  if [ "$name" = "c2" ]; then
    ncu -i $rep.ncu-rep --page source --csv --kernel-name regex:k_fwd_seq > gpurun_out/${tag}_source_c2_fwd.csv 2>/dev/null
  else
    rm -f $rep.ncu-rep
  fi
done
ls -la gpurun_out | tail -20
