# round-2 batch bd: no per-super-tile "fresh" vote once the warp has a max
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_bd.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_prevhm.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_bd.log 2>&1
