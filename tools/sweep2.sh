#!/bin/bash
for m in 0 1 2 3; do
  echo "== nochain=$m"; PDSSM_DEBUG_NOCHAIN=$m TAU=32 timeout 100 python tools/diag_paths.py 2>&1 | grep auto | head -1
done
