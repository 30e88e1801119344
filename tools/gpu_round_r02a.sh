set -x
python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/gpu_tests.log
python tools/parity.py --out gpurun_out/PARITY_r02.json > gpurun_out/parity.log 2>&1
python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
for dd in 0.1 0.125 0.25 0.5; do python bench.py --workload hunyuan --density $dd --no-e2e --no-cpu > gpurun_out/sweep_hunyuan_$dd.json 2>gpurun_out/sweep_hunyuan_$dd.err; done
