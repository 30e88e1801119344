# round-2 batch ac: host-path pipeline chunk count sweep (PISA_B200_HOST_CHUNKS) on the e2e number
for r in 1 2; do for c in 4 6 8 10 13 16 20 26; do
  PISA_B200_HOST_CHUNKS=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('chunks=$c', 'e2e_ms', round(j['e2e']['ms_per_step'],3), 'dev_ms', round(j['ms_per_step'],3))" >> gpurun_out/ab_hostchunks.log 2>&1
done; done
