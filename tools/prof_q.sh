set -x
bash tools/prof_fwd_src.sh q1
for r in smsp__pcsamp_warps_issue_stalled_long_scoreboard smsp__pcsamp_warps_issue_stalled_short_scoreboard smsp__pcsamp_warps_issue_stalled_wait smsp__pcsamp_warps_issue_stalled_selected; do
python tools/ncu_stall_by_reason.py gpurun_out/prof_q1.ncu-rep k_fwd_seq $r 30 > gpurun_out/q1_$r.txt 2>&1; done
ncu -i gpurun_out/prof_q1.ncu-rep --page source --csv --print-source sass > gpurun_out/q1_sass.csv 2>/dev/null
head -3 gpurun_out/q1_sass.csv | cut -c1-600
rm -f gpurun_out/prof_q1.ncu-rep
gzip -f gpurun_out/q1_sass.csv
