# round-2 batch i: K/V stage split of the fused kernel (3K+3V vs 2K+4V), both routings
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_k2v4.so gaussian clustered > gpurun_out/ab_k3_i.log 2>&1
