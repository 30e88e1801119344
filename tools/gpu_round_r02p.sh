# round-2 batch p: head-chunked two-kernel select (keys L2-resident) -- chunk size A/B
for r in 1 2; do
for mb in 0 20 40 80; do
  PISA_B200_SELECT_CHUNK_MB=$mb timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('chunk_mb=$mb', round(j['ms_per_step'],3), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])" >> gpurun_out/ab_select_p.log 2>&1
done; done
timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or plan or parity or router or cov" 2>&1 | tail -3 >> gpurun_out/ab_select_p.log
