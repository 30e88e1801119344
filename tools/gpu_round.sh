#!/bin/bash
# One GPU session: tests, bench (JSON), launch list, ncu captures of the kernels.
# Usage (under gpurun): bash tools/gpu_round.sh TAG
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_attn|block_stats|score_kernel|topk_kernel" -s 4 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log
head -c 2500 gpurun_out/bench_$TAG.json
