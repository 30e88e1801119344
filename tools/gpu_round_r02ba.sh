# round-2 batch ba: racecheck after the persistent K1's all-thread mbarrier arrives; K1 tests; K1 timing
set -x
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py --quick > gpurun_out/san_racecheck2.log 2>&1
grep -E "RACECHECK SUMMARY|calls" gpurun_out/san_racecheck2.log > gpurun_out/san_summary2.log
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "prepare or stats or hbar or norms or fused_matches" 2>&1 | tail -2 >> gpurun_out/san_summary2.log
for r in 1 2; do timeout 300 python bench.py --steps 10 --no-e2e --no-cpu --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print(round(j['ms_per_step'],3), 'K1', round(k['block_stats_kernel']['ms_per_launch'],4), j['hbm_rooflines']['block_stats_kernel']['frac'])" >> gpurun_out/san_summary2.log; done
