# round-2 batch ae: MMA warp event loop (PV_{g+1} no longer waits behind S_{g+3}'s K tile); + nanosleep variant
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ae.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_prevlist.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_ae.log 2>&1
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_evns.so gaussian clustered >> gpurun_out/ab_k3_ae.log 2>&1
for d in clustered gaussian; do
  PISA_B200_LIB=$L/libpisa_b200_trace.so timeout 300 python tools/trace_timeline.py 40 $d > gpurun_out/trace_ev_$d.txt 2>&1
done
