# round-2 batch k: top-k radix early exit (smem form) and register-form bucket limit
set -x
L=paper_2602_01077_b200/lib
for v in "" te0 treg40; do
  echo "== ${v:-base}" >> gpurun_out/gpu_tests_k.log
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or plan or tie or force or golden or covariance" 2>&1 | tail -3 >> gpurun_out/gpu_tests_k.log
done
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for v in "" te0 treg40; do
    lib=$L/libpisa_b200${v:+_$v}.so
    PISA_B200_LIB=$lib timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan ${v:-base}" >> gpurun_out/ab_topk_k.log 2>&1
    for w in hunyuan flux; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "$w ${v:-base}" >> gpurun_out/ab_topk_k.log 2>&1
    done
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_k.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
