# round-2 batch ar: K1b forked beside the select, not under stream capture
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ar.log
L=$PWD/paper_2602_01077_b200/lib
for r in 1 2; do for lib in libpisa_b200_nofork.so libpisa_b200.so; do for w in flux sd35; do
  PISA_B200_LIB=$L/$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$lib $w', round(j['ms_per_step'],4), 'graph', round(j['graph']['ms_per_step'],4))" >> gpurun_out/ab_fork_ar.log 2>&1
done; done; done
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_nofork.so $L/libpisa_b200.so gaussian >> gpurun_out/ab_fork_ar.log 2>&1
