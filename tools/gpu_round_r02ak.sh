# round-2 batch ak: prologue of head chunk c+1 on a high-priority side stream during the fused kernel of chunk c
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/gpu_tests_ak.log
for r in 1 2; do for nc in 0 2 4 8; do
  PISA_B200_OVERLAP_CHUNKS=$nc timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('chunks=$nc', round(j['ms_per_step'],3), {n:round(v['ms_per_launch'],3) for n,v in k.items()}, j['gpu_launches'], j['clocks']['sm_mhz'])" >> gpurun_out/ab_ovl_ak.log 2>&1
done; done
for nc in 0 4; do
  PISA_B200_OVERLAP_CHUNKS=$nc timeout 300 python bench.py --steps 10 --data clustered --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('clustered chunks=$nc', round(j['ms_per_step'],3), j['clocks']['sm_mhz'])" >> gpurun_out/ab_ovl_ak.log 2>&1
done
