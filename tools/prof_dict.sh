#!/bin/bash
# surrogate-gradient check: GPU tests, bench figures, ncu of the dictionary-gradient kernel
mkdir -p gpurun_out
TAG=${1:-d1}
timeout 600 python -m pytest tests/test_gpu_surrogate.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b.json
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value']/1e6, json.dumps(d['layer_kernels']['surrogate_grads']))"
ncu --set full --clock-control none --import-source on -k regex:"k_dict_grad_tc" -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep k_dict_grad > gpurun_out/ncu_summary_dict_${TAG}.txt 2>&1
grep -E "Duration|DRAM Through|Issue Slots|dram__bytes|stall" gpurun_out/ncu_summary_dict_${TAG}.txt
