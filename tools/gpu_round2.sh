#!/bin/bash
TAG=${1:-r}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --data clustered --no-e2e --no-cpu > gpurun_out/bench_${TAG}_clustered.json 2>> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_attn|block_stats|score_kernel|topk_kernel" -s 4 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_$TAG.log 2>&1
for f in gpurun_out/bench_$TAG.json gpurun_out/bench_${TAG}_clustered.json; do python -c "
import json,sys; j=json.load(open('$f')); print('$f', 'ms', round(j['ms_per_step'],3), 'TF', round(j['value']), 'frac', round(j['roofline']['frac'],3), 'exec', round(j['roofline']['executed_frac'],3), 'U/k', round(j['roofline']['union_over_k'],3), {k:round(v['ms_per_launch'],3) for k,v in j['kernels'].items()}, 'dense', j['dense_baseline'] and round(j['dense_baseline']['ms'],1), 'e2e', j['e2e'] and round(j['e2e']['ms_per_step'],1), 'cpu', j['cpu_baseline'] and j['cpu_baseline'].get('value'), j['clocks'])"; done
