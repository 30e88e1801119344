#!/bin/bash
# Builds paper_2602_01077_b200/lib/libpisa_b200_<name>.so: the library with one
# source recompiled under extra -D flags (A/B of compile-time switches).
#   bash tools/build_flag_variant.sh <name> <source.cu> "<flags>"
set -e
NAME=$1; SRC=$2; FLAGS=$3
cd /root/repo/paper_2602_01077_b200
python -c "import sys; sys.path.insert(0, '..'); from paper_2602_01077_b200 import build as b; b.build()" > /dev/null
OD=lib/obj_$NAME; rm -rf $OD; mkdir -p $OD
cp lib/obj/*.o $OD/
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr $FLAGS -I csrc -I ../include -c csrc/$SRC -o $OD/${SRC%.cu}.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o lib/libpisa_b200_$NAME.so $OD/*.o
echo lib/libpisa_b200_$NAME.so
