# round-2 batch h: single-pass softmax + MUFU ping-pong K3 -- parity subset, A/B, traces
set -x
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -k "fused or golden or randomized or variant or diag or ragged or overflow or finite" 2>&1 | tail -15 > gpurun_out/gpu_tests_h.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_h.log 2>&1
timeout 600 bash tools/ab_lib.sh $L/libpisa_b200_nopp.so $L/libpisa_b200.so gaussian clustered >> gpurun_out/ab_k3_h.log 2>&1
for d in clustered gaussian; do
  PISA_B200_LIB=$L/libpisa_b200_trace.so timeout 300 python tools/trace_timeline.py 40 $d > gpurun_out/trace_new_$d.txt 2>&1
done
