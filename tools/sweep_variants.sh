#!/bin/bash
# usage: TAUS="32 64" bash tools/sweep_variants.sh VARIANT... (strict fused path)
for v in "$@"; do
 for tau in ${TAUS:-32 64}; do
  echo "== $v tau=$tau $(PDSSM_PATH=fused PDSSM_LIB_VARIANT=$v TAU=$tau timeout 100 python tools/diag_paths.py 2>&1 | grep -E '^fused|rror' | head -1)"
 done
done
