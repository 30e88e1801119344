# round-2 batch h: streamed select (score via the pipelined kernel + topk_kernel)
# and top-k variants (match_any-aggregated digit counts, batched row loads)
set -x
L=paper_2602_01077_b200/lib
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select or plan or tie or force" 2>&1 | tail -5 > gpurun_out/gpu_tests_h.log
for v in tk1 tk2 tl8 tk1l8 tk2l8; do
  echo "== $v" >> gpurun_out/gpu_tests_h.log
  PISA_B200_LIB=$L/libpisa_b200_$v.so timeout 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "select" 2>&1 | tail -2 >> gpurun_out/gpu_tests_h.log
done
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for fs in 0 stream; do
    if [ $fs = stream ]; then unset PISA_B200_FUSED_SELECT; else export PISA_B200_FUSED_SELECT=$fs; fi
    timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan fs=$fs" >> gpurun_out/ab_sel_h.log 2>&1
  done
  unset PISA_B200_FUSED_SELECT
  for v in tk1 tk2 tl8 tk1l8 tk2l8; do
    PISA_B200_LIB=$L/libpisa_b200_$v.so timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | sel "wan stream $v" >> gpurun_out/ab_sel_h.log 2>&1
  done
  for w in flux sd35; do
    for v in "" tk1 tk2 tl8 tk1l8; do
      lib=$L/libpisa_b200${v:+_$v}.so
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "$w ${v:-base}" >> gpurun_out/ab_sel_h.log 2>&1
    done
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
