#!/bin/bash
# build libpdssm.so variants with different fused-kernel constants into paper_2605_19150_b200/variants/
mkdir -p paper_2605_19150_b200/variants
build() { # name, defines
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Xptxas -v $2 \
    -o paper_2605_19150_b200/variants/$1.so paper_2605_19150_b200/csrc/pdssm_api.cu > /tmp/ptx_$1.txt 2>&1
  echo "built $1: $(grep -A2 'k_fwd_fusedIfLi2ELi4ELb0' /tmp/ptx_$1.txt | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ') / $(grep -A2 'k_bwd_fusedIffLi2ELi4ELb0' /tmp/ptx_$1.txt | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
}
build v_f14g2p2_b13g1p3 "-DPDSSM_WARPS_FWD=14 -DPDSSM_G_FWD=2 -DPDSSM_PF_FWD=2 -DPDSSM_WARPS_BWD=13 -DPDSSM_G_BWD=1 -DPDSSM_PF_BWD=3" &
build v_f16g2p2_b12g2p2 "-DPDSSM_WARPS_FWD=16 -DPDSSM_G_FWD=2 -DPDSSM_PF_FWD=2 -DPDSSM_WARPS_BWD=12 -DPDSSM_G_BWD=2 -DPDSSM_PF_BWD=2" &
build v_f12g4p1_b14g1p2 "-DPDSSM_WARPS_FWD=12 -DPDSSM_G_FWD=4 -DPDSSM_PF_FWD=1 -DPDSSM_WARPS_BWD=14 -DPDSSM_G_BWD=1 -DPDSSM_PF_BWD=2" &
wait
