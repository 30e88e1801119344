# round-2 measurement batch b: tests on the new default library, microbenchmark,
# K1 and exp2-split A/B, bench line, ncu launch list + --set full capture
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests_b.log
./tools/st_mix > gpurun_out/st_mix.log 2>&1
bash tools/ab_k1.sh > gpurun_out/ab_k1.log 2>&1
bash tools/ab_poly.sh b00 b11 b55 > gpurun_out/ab_poly.log 2>&1
python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_stats_persistent|score_kernel|topk_kernel|fused_attn" -s 8 -c 4 -o gpurun_out/prof_r02b python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_r02b.log 2>&1
