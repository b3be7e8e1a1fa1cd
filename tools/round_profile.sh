#!/bin/bash
# Round artefacts: bench line, ncu launch list of the bench command, full ncu capture of the two
# scan kernels (-> dram traffic per launch) and of the tensor-core GEMM (projection).
set -x
mkdir -p gpurun_out
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu_${TAG}.txt
ncu --set full --clock-control none --import-source on -k regex:"k_(fwd|bwd)_(fused|seq)" -s 2 -c 2 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-layer > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/prof_${TAG}.ncu-rep profiles/traffic_latest.json
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep k_fwd_ > gpurun_out/ncu_summary_fwd_${TAG}.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep k_bwd_ > gpurun_out/ncu_summary_bwd_${TAG}.txt 2>&1
cp profiles/traffic_latest.json gpurun_out/traffic_${TAG}.json
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc" -c 3 \
    -o gpurun_out/prof_gemm_${TAG} python tools/time_gemm.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_gemm_${TAG}.ncu-rep k_gemm_tc > gpurun_out/ncu_summary_gemm_${TAG}.txt 2>&1
ls -la gpurun_out
# keep gpurun_out under the 64 MiB copy-back limit
rm -f gpurun_out/prof_gemm_${TAG}.ncu-rep
du -sh gpurun_out
# NEXT-1 dictionary-gradient kernel (tcgen05 3xTF32 grouped outer products)
ncu --set full --clock-control none --import-source on -k regex:"k_dict_grad_tc" -c 1 \
    -o gpurun_out/prof_dict_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_dict_${TAG}.ncu-rep k_dict_grad > gpurun_out/ncu_summary_dict_${TAG}.txt 2>&1
rm -f gpurun_out/prof_dict_${TAG}.ncu-rep
du -sh gpurun_out
rm -f gpurun_out/prof_${TAG}.ncu-rep
du -sh gpurun_out
