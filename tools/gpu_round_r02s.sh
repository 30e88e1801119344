# round-2 batch s: single-pass (speculative-max) softmax in the production kernel; with 2 K + 3 V stages
set -x
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "fused or golden or randomized or variant or diag or ragged or overflow or finite or qrange or pairing" 2>&1 | tail -3 > gpurun_out/gpu_tests_s.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1500 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_s.log 2>&1
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200_spk2v3.so gaussian clustered >> gpurun_out/ab_k3_s.log 2>&1
