# round-2 batch ax: one exp code path when the MUFU/FMA splits agree
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ax.log
L=$PWD/paper_2602_01077_b200/lib
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_both.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_both_ax.log 2>&1
