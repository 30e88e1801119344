# round-2 batch ah: full GPU suite + bench on the new default (single-pass softmax, union list, no prefetch)
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests_ah.log
python bench.py --no-cpu --no-e2e > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err
python bench.py --data clustered --no-cpu --no-e2e > gpurun_out/bench_r02h_clustered.json 2> /dev/null
