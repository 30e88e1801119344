# round-2 batch s: ncu --set full of the full-range pairing kernels
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense"
for k in overlap_tc_kernel cand_full_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/r02s_$k $B > /dev/null 2>&1
done
