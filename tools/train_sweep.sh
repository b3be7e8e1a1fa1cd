#!/bin/bash
# NEXT-4 desk-scale FSA training sweep (run under gpurun); one JSON line per run
tag=${1:-r02}
out=gpurun_out/${tag}_train_sweep.jsonl; rm -f $out
for args in "--steps 6000" "--steps 6000 --t0 0.5 --t1 0.05" "--steps 6000 --t0 2.0 --t1 0.2" "--steps 6000 --bmag 4"; do
  timeout 900 python -m paper_2605_19150_b200.train_fsa --tasks parity,cycle_nav,even_pairs,mod_arith $args >> $out 2>> gpurun_out/${tag}_train_sweep.err
done
echo sweep $?
