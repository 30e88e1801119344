# round-2 batch ab: single-pass softmax + M=64 PV for single-use key blocks (power) vs production
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_k3_spec_m64pv.so gaussian clustered > gpurun_out/ab_k3_ab.log 2>&1
PISA_B200_LIB=$L/libpisa_b200_k3_spec_m64pv.so timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "fused or golden or randomized or variant or diag or ragged or overflow or finite or qrange or pairing" 2>&1 | tail -2 >> gpurun_out/ab_k3_ab.log
