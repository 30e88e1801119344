# round-2 batch p: final code -- default bench line, clustered, image sizes and Wan2.1-1.3B (K1 chunking), GPU tests
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests_r02p.log
python bench.py > gpurun_out/bench_r02p.json 2> gpurun_out/bench_r02p.err
python bench.py --data clustered --no-cpu > gpurun_out/bench_r02p_clustered.json 2> /dev/null
for w in flux sd35 wan13b; do python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/sweep_r02p_$w.json 2>/dev/null; done
