# round-2 batch o: racecheck after the top-k early-exit fix; pair_match with staged candidates (base) vs plain (pm0):
# identical outputs (hashes) and timing
set -x
L=paper_2602_01077_b200/lib
timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize.py --quick > gpurun_out/sanitize_r02o_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_r02o_racecheck.log
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or pairing or tie" 2>&1 | tail -2 > gpurun_out/gpu_tests_o.log
for v in "" pm0; do
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 600 python tools/hash_outputs.py > gpurun_out/hash_o_${v:-base}.log 2>&1
done
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for v in "" pm0; do
    PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan ${v:-base}" >> gpurun_out/ab_pair_o.log 2>&1
    PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 300 python bench.py --data clustered --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan-clustered ${v:-base}" >> gpurun_out/ab_pair_o.log 2>&1
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_o.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
