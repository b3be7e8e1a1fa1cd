#!/bin/bash
# Round-end evidence on one GPU: the GPU test suite, every bench line (tools/bench_all.sh), the default
# launch list and the per-config ncu summaries (tools/prof_final.sh).  Output under gpurun_out/.
tag=${1:-r02w}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/${tag}_pytest_gpu.txt
bash tools/bench_all.sh $tag > gpurun_out/${tag}_bench_all.log 2>&1
bash tools/prof_final.sh $tag > gpurun_out/${tag}_prof.log 2>&1
