# round-2 batch ay: TMA boxes issued one per lane (Q by warp 1 at kernel start; K 4 lanes; V 2 lanes)
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ay.log
L=$PWD/paper_2602_01077_b200/lib
PISA_B200_LIB=$L/libpisa_b200_trace.so timeout 300 python tools/trace_timeline.py 40 gaussian > gpurun_out/trace_tma_gaussian.txt 2>&1
for r in 1 2; do for lib in libpisa_b200_g.so libpisa_b200.so; do for w in flux sd35; do
  PISA_B200_LIB=$L/$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$lib $w', round(j['ms_per_step'],4), 'graph', round(j['graph']['ms_per_step'],4), 'K3', round(k['fused_attn_kernel']['ms_per_launch'],4))" >> gpurun_out/ab_tma_ay.log 2>&1
done; done; done
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_g.so $L/libpisa_b200.so gaussian clustered >> gpurun_out/ab_tma_ay.log 2>&1
