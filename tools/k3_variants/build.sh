#!/bin/bash
# Builds paper_2602_01077_b200/lib/libpisa_b200_<variant>.so: the library with
# K3 replaced by tools/k3_variants/<variant>.cu (A/B with tools/ab_lib.sh).
#   bash tools/k3_variants/build.sh k3_rowthread [EXTRA_NVCC_FLAGS]
set -e
V=$1; EXTRA=$2
cd /root/repo/paper_2602_01077_b200
python -c "import sys; sys.path.insert(0, '..'); from paper_2602_01077_b200 import build as b; b.build()" > /dev/null
OD=lib/obj_$V; mkdir -p $OD
cp lib/obj/*.o $OD/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr $EXTRA -I csrc -I ../include -c ../tools/k3_variants/$V.cu -o $OD/k3_fused_attn.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o lib/libpisa_b200_$V.so $OD/*.o
echo lib/libpisa_b200_$V.so
