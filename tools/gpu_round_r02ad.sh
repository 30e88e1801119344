# round-2 batch ad: per-CTA union list in shared memory (one load per super-tile instead of a bitmask walk per role)
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ad.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_prevlist.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_ad.log 2>&1
for d in clustered gaussian; do
  PISA_B200_LIB=$L/libpisa_b200_trace.so timeout 300 python tools/trace_timeline.py 40 $d > gpurun_out/trace_list_$d.txt 2>&1
done
