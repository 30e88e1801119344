# round-2 batch m: K1 H partial with 32-byte stores (base) vs 16-byte (k1s0); FLUX K1 chunk size
set -x
L=paper_2602_01077_b200/lib
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "prepare or stats or golden or hbar" 2>&1 | tail -3 > gpurun_out/gpu_tests_m.log
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for v in "" k1s0; do
    lib=$L/libpisa_b200${v:+_$v}.so
    for w in flux sd35 wan14b hunyuan; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --steps 5 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "$w ${v:-base}" >> gpurun_out/ab_k1_m.log 2>&1
    done
  done
  for g in 4 6 8 12; do
    PISA_B200_STATS_G=$g timeout 300 python bench.py --workload flux --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "flux G=$g" >> gpurun_out/ab_k1_m.log 2>&1
    PISA_B200_STATS_G=$g timeout 300 python bench.py --workload sd35 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "sd35 G=$g" >> gpurun_out/ab_k1_m.log 2>&1
  done
done
