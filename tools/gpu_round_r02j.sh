# round-2 batch j: register-resident top-k (topk_reg_kernel) vs the shared-memory topk_kernel
set -x
L=paper_2602_01077_b200/lib
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or plan or tie or force or golden or covariance" 2>&1 | tail -3 > gpurun_out/gpu_tests_j.log
timeout 1200 python tools/parity.py --configs smoke,flux,wan14b,hunyuan --densities 0.125 --out gpurun_out/parity_j.json > gpurun_out/parity_j.log 2>&1
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for v in "" treg0; do
    lib=$L/libpisa_b200${v:+_$v}.so
    PISA_B200_LIB=$lib timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan ${v:-reg}" >> gpurun_out/ab_topk_j.log 2>&1
    for w in flux sd35 hunyuan; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "$w ${v:-reg}" >> gpurun_out/ab_topk_j.log 2>&1
    done
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_j.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk_reg -c 1 -f -o gpurun_out/r02j_topk_reg python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
