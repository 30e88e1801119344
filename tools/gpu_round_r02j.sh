# round-2 batch j: M=64 MMAs for single-use key blocks (Q in TMEM) -- parity subset, A/B vs previous
set -x
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "fused or golden or randomized or variant or diag or ragged or overflow or finite or qrange or pairing" 2>&1 | tail -15 > gpurun_out/gpu_tests_j.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_j.log 2>&1
