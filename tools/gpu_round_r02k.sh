# round-2 batch k: where do the M=64 kernel's extra cycles come from? force-M128 timing variant
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_m128.so $L/libpisa_b200.so gaussian > gpurun_out/ab_k3_k.log 2>&1
