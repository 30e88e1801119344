# round-2 batch ap: fused select by default for short heads (image sizes)
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ap.log
for r in 1 2; do for fs in 0 auto; do for w in flux sd35; do
  if [ $fs = auto ]; then unset PISA_B200_FUSED_SELECT; else export PISA_B200_FUSED_SELECT=$fs; fi
  timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$w fused_select=$fs', round(j['ms_per_step'],4), 'graph', round(j['graph']['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()})" >> gpurun_out/ab_sel_ap.log 2>&1
done; done; done
unset PISA_B200_FUSED_SELECT
