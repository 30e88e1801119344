#!/bin/bash
# quick GPU iteration: correctness diag + bench (no e2e/cpu) + timeline
TAG=${1:-q}
timeout 300 python tools/gpu_diag.py > gpurun_out/diag_$TAG.log 2>&1; echo "diag OK count: $(grep -c ' OK' gpurun_out/diag_$TAG.log) FAIL: $(grep -c FAIL gpurun_out/diag_$TAG.log)"; grep -E "K3 hybrid" gpurun_out/diag_$TAG.log | head -4
timeout 300 python bench.py --no-e2e --no-cpu ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err
python -c "
import json; j=json.load(open('gpurun_out/bench_$TAG.json')); print('ms', round(j['ms_per_step'],3), 'TFLOPS', round(j['value']), 'frac', round(j['roofline']['frac'],3), 'exec', round(j['roofline']['executed_frac'],3), {k:round(v['ms_per_launch'],3) for k,v in j['kernels'].items()}, 'dense', round(j['dense_baseline']['ms'],2), j['clocks'])" || tail -5 gpurun_out/bench_$TAG.err
timeout 300 python tools/trace_timeline.py > gpurun_out/trace_$TAG.txt 2>&1; sed -n 1p gpurun_out/trace_$TAG.txt; sed -n 240,246p gpurun_out/trace_$TAG.txt; tail -1 gpurun_out/trace_$TAG.txt
