#!/bin/bash
# usage: buildvar.sh NAME "EXTRA_FLAGS"
set -e
cd /root/repo/paper_2602_01077_b200
NAME=$1; EXTRA=$2
OD=lib/obj_$NAME; mkdir -p $OD
for f in k1_block_stats k1c_block_norms k2_select k2p_pairing k3_fused_attn selftest_mma generate pisa_b200; do
  if [ "$f" = "k3_fused_attn" ] || [ ! -f $OD/$f.o ] || [ csrc/$f.cu -nt $OD/$f.o ] || [ csrc/kernels.h -nt $OD/$f.o ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr $EXTRA -I csrc -I ../include -c csrc/$f.cu -o $OD/$f.o
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o lib/libpisa_b200_$NAME.so $OD/*.o
