# round-2 batch as: K1 chunk size (key blocks per work item) and persistent vs one-chunk-per-CTA K1 at image sizes
L=$PWD/paper_2602_01077_b200/lib
for lib in libpisa_b200.so libpisa_b200_k1np.so; do for g in 4 8 12 18 24; do for w in flux sd35; do
  PISA_B200_STATS_G=$g PISA_B200_LIB=$L/$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$lib G=$g $w', round(j['ms_per_step'],4), 'graph', round(j['graph']['ms_per_step'],4), 'K1', round(k['block_stats_kernel']['ms_per_launch'],4), 'K1b', round(k['hbar_reduce_kernel']['ms_per_launch'],4))" >> gpurun_out/ab_k1_as.log 2>&1
done; done; done
