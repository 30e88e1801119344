# round-2 batch d: thread-per-row / alternating-warpgroup K3 -- parity subset,
# then A/B against the previous kernel (libpisa_b200_k3old.so) on both routings
set -x
timeout 600 python -m pytest tests/test_gpu.py -m gpu -x -q -k "fused or golden or randomized or variant or diag or ragged" 2>&1 | tail -15 > gpurun_out/gpu_tests_d.log
L=$PWD/paper_2602_01077_b200/lib
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_d.log 2>&1
