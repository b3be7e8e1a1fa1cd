#!/bin/bash
# NEXT-4: the Table 1 analogue with the settings the parity sweep selected (lr 5e-4, |D| init sigmoid(5))
tag=${1:-r02}
out=gpurun_out/${tag}_train_final.jsonl; rm -f $out
timeout 2400 python -m paper_2605_19150_b200.train_fsa --tasks parity,cycle_nav,even_pairs,mod_arith --steps 15000 \
  --lr 5e-4 --bmag 5 --seeds 2 >> $out 2>> gpurun_out/${tag}_train_final.err
echo train_final $?
