#!/bin/bash
# NEXT-4: parity-focused training variants (run under gpurun)
tag=${1:-r02}
out=gpurun_out/${tag}_train_parity.jsonl; rm -f $out
for args in "--steps 15000" "--steps 15000 --bmag 5" "--steps 15000 --t0 1.0 --t1 1.0 --bmag 5" "--steps 15000 --dict 4 --bmag 5" "--steps 15000 --lr 5e-4 --bmag 5"; do
  timeout 900 python -m paper_2605_19150_b200.train_fsa --tasks parity $args >> $out 2>> gpurun_out/${tag}_train_parity.err
done
echo parity sweep $?
