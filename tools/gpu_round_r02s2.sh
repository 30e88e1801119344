# round-2 re-entry confirmation on the restored tree: GPU tests, smoke, headline bench, clustered, image presets
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests_s2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s2.log
python bench.py > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err
python bench.py --data clustered --no-cpu > gpurun_out/bench_s2_clustered.json 2> gpurun_out/bench_s2_clustered.err
for w in flux sd35; do python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/sweep_s2_$w.json 2>/dev/null; python bench.py --workload $w --router covariance --no-cpu --no-e2e > gpurun_out/sweep_s2_${w}_covariance.json 2>/dev/null; done
