# round-2 batch bb: 16 softmax warps (two per row set, 16 columns per thread) vs 8
set -x
PISA_B200_LIB=$PWD/paper_2602_01077_b200/lib/libpisa_b200_w16.so timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_bb.log
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "fused or golden or randomized" 2>&1 | tail -2 >> gpurun_out/gpu_tests_bb.log
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_w8.so $L/libpisa_b200_w16.so gaussian clustered > gpurun_out/ab_w16_bb.log 2>&1
for lib in libpisa_b200_w8.so libpisa_b200_w16.so; do for w in flux sd35; do
  PISA_B200_LIB=$L/$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$lib $w', round(j['ms_per_step'],4), 'K3', round(k['fused_attn_kernel']['ms_per_launch'],4))" >> gpurun_out/ab_w16_bb.log 2>&1
done; done
