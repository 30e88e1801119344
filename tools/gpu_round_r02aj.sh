# round-2 batch aj: 3 K stages again (with the union list + single pass); softmax waits with nanosleep backoff
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_ks3.so gaussian clustered > gpurun_out/ab_k3_aj.log 2>&1
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_sp2.so gaussian clustered >> gpurun_out/ab_k3_aj.log 2>&1
