#!/bin/bash
# per-step cost and fixed (prologue) cost of the single-chunk kernels: config-2 shape over L
for L in 128 256 512 1024 2048; do echo "L=$L"; python tools/time_cfg.py 16 8 $L 128 32 2 f32 auto; done
