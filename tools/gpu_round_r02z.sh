# round-2 batch z: candidate kernel with paired 4-byte overlap loads
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), 'U/k', round(j['roofline']['union_over_k'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "pairing or range" 2>&1 | tail -2 > gpurun_out/gpu_tests_z.log
timeout 600 python tools/hash_outputs.py > gpurun_out/hash_z.log 2>&1
timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan" >> gpurun_out/ab_z.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_z.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
