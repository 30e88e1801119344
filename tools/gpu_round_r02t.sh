# round-2 batch t: overlap_tc v2 (no staging, 256 threads, 3 CTAs/SM) + top-4 candidate pop; equality vs int8 mma.sync (otc0); full vs window
set -x
L=paper_2602_01077_b200/lib
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "pairing" 2>&1 | tail -3 > gpurun_out/gpu_tests_t.log
for v in "" otc0; do
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 600 python tools/hash_outputs.py > gpurun_out/hash_t_${v:-base}.log 2>&1
done
PISA_B200_PAIR_FULL=0 timeout 600 python tools/hash_outputs.py > gpurun_out/hash_t_window.log 2>&1
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), 'U/k', round(j['roofline']['union_over_k'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for f in 1 0; do
    PISA_B200_PAIR_FULL=$f timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan full=$f" >> gpurun_out/ab_pair_t.log 2>&1
    PISA_B200_PAIR_FULL=$f timeout 300 python bench.py --data clustered --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan-clustered full=$f" >> gpurun_out/ab_pair_t.log 2>&1
    PISA_B200_PAIR_FULL=$f timeout 300 python bench.py --workload hunyuan --steps 5 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "hunyuan full=$f" >> gpurun_out/ab_pair_t.log 2>&1
    PISA_B200_PAIR_FULL=$f timeout 300 python bench.py --workload wan13b --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan13b full=$f" >> gpurun_out/ab_pair_t.log 2>&1
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_t.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"overlap_tc|cand_full" -c 2 -f -o gpurun_out/r02t_pair python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
