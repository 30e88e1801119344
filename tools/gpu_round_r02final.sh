# round-2 final-code check: full GPU suite, smoke, default bench line (+ clustered), launch list
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --data clustered --no-cpu > gpurun_out/bench_final_clustered.json 2> /dev/null
python bench.py --workload hunyuan --no-cpu --no-e2e > gpurun_out/sweep_final_hunyuan.json 2> /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
