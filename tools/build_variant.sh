#!/bin/bash
# build libpdssm.so variants with different fused-kernel constants into paper_2605_19150_b200/variants/
# usage: bash tools/build_variant.sh NAME "DEFINES" [NAME "DEFINES" ...]
mkdir -p paper_2605_19150_b200/variants
build() { # name, defines
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v $2 \
    -o paper_2605_19150_b200/variants/$1.so paper_2605_19150_b200/csrc/pdssm_api.cu > /tmp/ptx_$1.txt 2>&1
  echo "built $1: $(grep -A2 'k_fwd_seqIfLi2ELb0ELb0ELb0ELi128E' /tmp/ptx_$1.txt | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ') / $(grep -A2 'k_bwd_seqIffLi2ELb0ELi128E' /tmp/ptx_$1.txt | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
}
while [ $# -ge 2 ]; do build "$1" "$2" & shift 2; done
wait
