# round-2 batch aw: Phase-2 ragged-block p picked once (not a select per element)
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_aw.log
L=$PWD/paper_2602_01077_b200/lib
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_plold.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_pl_aw.log 2>&1
