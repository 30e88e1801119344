# round-2 batch aa: top-k first digit adapted to the row's common high bits (base) vs fixed top byte (ta0)
L=paper_2602_01077_b200/lib
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or tie or plan or golden or covariance" 2>&1 | tail -2 > gpurun_out/gpu_tests_aa.log
timeout 1200 python tools/parity.py --configs smoke,flux,wan14b --densities 0.125 --out gpurun_out/parity_aa.json > gpurun_out/parity_aa.log 2>&1
for r in 1 2; do for v in "" ta0; do
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan ${v:-adapt}" >> gpurun_out/ab_aa.log 2>&1
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 300 python bench.py --workload hunyuan --steps 5 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "hunyuan ${v:-adapt}" >> gpurun_out/ab_aa.log 2>&1
done; done
for v in "" ta0; do
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk -c 4 --csv --log-file gpurun_out/launches_aa_${v:-adapt}.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
done
