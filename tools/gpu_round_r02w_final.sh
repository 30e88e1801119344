# round-2 measurement batch w (final code: full-range pairing search by default, overlap on tcgen05 kind::i8):
# GPU tests + smoke, bench line, every BASELINE config vs dense, Hunyuan density sweep, parity vs the
# reference, ncu launch list + --set full capture, compute-sanitizer
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gpu_tests_r02w.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02w.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r02w.log
python bench.py > gpurun_out/bench_r02w.json 2> gpurun_out/bench_r02w.err
python bench.py --data clustered --no-cpu > gpurun_out/bench_r02w_clustered.json 2> gpurun_out/bench_r02w_clustered.err
python bench.py --router covariance --no-cpu --no-e2e > gpurun_out/bench_r02w_covariance.json 2> /dev/null
for w in flux sd35 wan13b hunyuan; do python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/sweep_r02w_$w.json 2>/dev/null; done
for w in flux sd35; do python bench.py --workload $w --router covariance --no-cpu --no-e2e > gpurun_out/sweep_r02w_${w}_covariance.json 2>/dev/null; done
for dd in 0.1 0.25 0.5; do python bench.py --workload hunyuan --density $dd --no-e2e --no-cpu > gpurun_out/sweep_r02w_hunyuan_d$dd.json 2>/dev/null; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02w_reference.json 2> gpurun_out/bench_r02w_reference.err
python tools/parity.py --out gpurun_out/PARITY_r02w.json > gpurun_out/parity_r02w.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02w.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_stats_persistent|select_fused|topk_kernel|fused_attn|overlap_tc|cand_full" -s 12 -c 6 -o gpurun_out/prof_r02w python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_r02w.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  q=--quick; [ $tool = memcheck ] && q=
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py $q > gpurun_out/sanitize_r02w_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_r02w_$tool.log
done
