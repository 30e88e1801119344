# round-2 batch ab: register-resident top-k with a register cap (8 / 6 CTAs per SM) at Wan2.1-14B
L=paper_2602_01077_b200/lib
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for v in tr40b8 tr40b6; do
  PISA_B200_LIB=$L/libpisa_b200_$v.so timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or tie" 2>&1 | tail -1 >> gpurun_out/gpu_tests_ab.log
done
for r in 1 2; do for v in "" tr40b8 tr40b6; do
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan ${v:-base}" >> gpurun_out/ab_ab.log 2>&1
done; done
for v in "" tr40b8 tr40b6; do
  PISA_B200_LIB=$L/libpisa_b200${v:+_$v}.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk -c 4 --csv --log-file gpurun_out/launches_ab_${v:-base}.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
done
