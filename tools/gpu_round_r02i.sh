# round-2 batch i: ncu --set full of topk_kernel, pair_candidates_kernel, pair_match_kernel (Wan2.1-14B)
# and block_stats_persistent_kernel at FLUX
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense"
for k in topk_kernel pair_candidates_kernel pair_match_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/r02i_$k $B > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_stats_persistent -c 1 -f -o gpurun_out/r02i_k1_flux $B --workload flux > /dev/null 2>&1
ls -la gpurun_out/
