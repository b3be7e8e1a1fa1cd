#!/bin/bash
for tau in 16 24 32 64; do
  echo "== tau=$tau"; TAU=$tau timeout 100 python tools/diag_paths.py 2>&1 | grep -A1 fused | head -2
done
