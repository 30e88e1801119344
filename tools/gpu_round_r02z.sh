# round-2 batch z: A/B of the committed kernel against the round-start kernel, image sizes
L=$PWD/paper_2602_01077_b200/lib
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200_k3old.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_k3_z.log 2>&1
for w in flux sd35; do for lib in libpisa_b200_k3old.so libpisa_b200.so; do
  PISA_B200_LIB=$L/$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$lib', '$w', round(j['ms_per_step'],4), 'fused', round(k['fused_attn_kernel']['ms_per_launch'],4), 'graph', round(j['graph']['ms_per_step'],4), 'dense', round(j['dense_baseline']['ms'],4), j['clocks'])" >> gpurun_out/ab_k3_z.log 2>&1
done; done
