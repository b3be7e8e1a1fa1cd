#!/bin/bash
# usage: TAU=.. bash tools/quick_prof.sh TAG : dram bytes + duration + instructions of the fused kernels
TAG=${1:-q}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:"k_(fwd|bwd)_fused" -s 2 -c 2 --csv --log-file gpurun_out/qp_${TAG}.csv python tools/diag_paths.py > /dev/null 2>&1
python tools/qp_parse.py gpurun_out/qp_${TAG}.csv
