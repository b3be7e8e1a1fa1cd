#!/bin/bash
for v in v_f14g2p2_b13g1p3 v_f16g2p2_b12g2p2 v_f12g4p1_b14g1p2; do
 for tau in 16 32 64; do
  echo "== $v tau=$tau $(PDSSM_LIB_VARIANT=$v TAU=$tau timeout 100 python tools/diag_paths.py 2>&1 | grep auto | head -1)"
 done
done
