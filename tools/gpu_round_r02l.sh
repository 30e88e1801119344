# round-2 batch l: previous fused kernel with 2 K + 3 V stages (frees 32 KB for a second Q image)
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200_k2v3.so gaussian clustered > gpurun_out/ab_k3_l.log 2>&1
