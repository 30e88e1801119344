# round-2 batch am: MMA issuer on warp 3 instead of warp 1 (the softmax warps q4 = 1 lag by ~1700 cycles on clustered routing)
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_mma3.so gaussian clustered > gpurun_out/ab_k3_am.log 2>&1
PISA_B200_LIB=$L/libpisa_b200_mma3tr.so timeout 300 python tools/trace_timeline.py 40 clustered > gpurun_out/trace_mma3_clustered.txt 2>&1
PISA_B200_LIB=$L/libpisa_b200_mma3.so timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "fused or golden or randomized or variant" 2>&1 | tail -2 >> gpurun_out/ab_k3_am.log
