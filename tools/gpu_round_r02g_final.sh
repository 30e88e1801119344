# round-2 measurement batch g (union list, single pass, K1b fork, faster pairing): bench line, sweep of
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests_r02g.log
# every BASELINE config vs dense, Hunyuan density sweep, parity vs the reference,
# ncu launch list + --set full capture
set -x
python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err
python bench.py --data clustered --no-cpu > gpurun_out/bench_r02g_clustered.json 2> gpurun_out/bench_r02g_clustered.err
python bench.py --router covariance --no-cpu --no-e2e > gpurun_out/bench_r02g_covariance.json 2> /dev/null
for w in flux sd35 wan13b hunyuan; do python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/sweep_r02g_$w.json 2>/dev/null; done
for w in flux sd35; do python bench.py --workload $w --router covariance --no-cpu --no-e2e > gpurun_out/sweep_r02g_${w}_covariance.json 2>/dev/null; done
for dd in 0.1 0.25 0.5; do python bench.py --workload hunyuan --density $dd --no-e2e --no-cpu > gpurun_out/sweep_r02g_hunyuan_d$dd.json 2>/dev/null; done
python tools/parity.py --out gpurun_out/PARITY_r02g.json > gpurun_out/parity_r02g.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02g.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_stats_persistent|score_kernel|topk_kernel|fused_attn|pair_cand" -s 8 -c 5 -o gpurun_out/prof_r02g python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_r02g.log 2>&1
