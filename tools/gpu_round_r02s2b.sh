# round-2 re-entry batch b (final code): parity vs the reference at every BASELINE config,
# reference arm, Hunyuan density sweep, ncu launch list + --set full capture of the headline step
set -x
timeout 1500 python tools/parity.py --out gpurun_out/PARITY_r02s2.json > gpurun_out/parity_r02s2.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02s2_reference.json 2> gpurun_out/bench_r02s2_reference.err
for dd in 0.1 0.125 0.25 0.5; do python bench.py --workload hunyuan --density $dd --no-e2e --no-cpu > gpurun_out/sweep_r02s2_hunyuan_d$dd.json 2>/dev/null; done
python bench.py --workload wan13b --no-cpu --no-e2e > gpurun_out/sweep_r02s2_wan13b.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02s2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_stats_persistent|select_fused|topk_kernel|fused_attn|overlap_tc|cand_full" -s 12 -c 6 -o gpurun_out/prof_r02s2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/ncu_r02s2.log 2>&1
