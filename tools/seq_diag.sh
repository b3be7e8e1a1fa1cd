#!/bin/bash
for v in "$@"; do echo "== $v $(PDSSM_LIB_VARIANT=$v PATHS=seq timeout 100 python tools/diag_paths.py 2>&1 | grep -E '^seq|rror' | head -1)"; done
