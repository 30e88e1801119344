# round-2 batch ag: single-pass softmax (s) x S prefetch (p), 2 x 2
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ag.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_s0p0.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_ag.log 2>&1
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_s1p0.so $L/libpisa_b200_s0p1.so gaussian clustered >> gpurun_out/ab_k3_ag.log 2>&1
