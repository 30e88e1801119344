# round-2 batch ai: softmax code deduplication (one call site per sub-tile, no both-split variant)
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ai.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_prevdd.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_ai.log 2>&1
