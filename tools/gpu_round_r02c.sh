# round-2 batch c (re-entry): shared-memory port microbenchmark (modes 0-6,
# one process each), GPU tests, fused vs two-kernel select, bench line
set -x
for m in 0 1 2 3 4 5 6; do timeout 60 ./tools/st_mix $m >> gpurun_out/st_mix_c.log 2>&1; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests_c.log
for fs in 1 0 1 0; do echo "fused_select=$fs" >> gpurun_out/ab_select_c.log; PISA_B200_FUSED_SELECT=$fs python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['ms_per_step'], {k:round(v['ms_per_launch'],4) for k,v in j['kernels'].items()}, j['clocks'])" >> gpurun_out/ab_select_c.log 2>&1; done
python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
python bench.py --data clustered --no-e2e --no-cpu > gpurun_out/bench_r02c_clustered.json 2> gpurun_out/bench_r02c_clustered.err
