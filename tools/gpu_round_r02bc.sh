# round-2 batch bc: the restored 8-warp kernel (dead prefetch code removed) -- tests and A/B vs the generalized one at 8 warps
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_bc.log
L=$PWD/paper_2602_01077_b200/lib
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_w8.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_bc.log 2>&1
