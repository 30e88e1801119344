#!/bin/bash
# K1 A/B: default library (persistent block statistics) vs k1old (one chunk per CTA)
cd /root/repo
for r in 1 2 3; do
  for L in paper_2602_01077_b200/lib/libpisa_b200.so paper_2602_01077_b200/lib/libpisa_b200_k1old.so; do
    PISA_B200_LIB=$PWD/$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; r=j['hbm_rooflines']; print('$(basename $L)', 'K1', round(k['block_stats_kernel']['ms_per_launch'],4), 'frac', round(r['block_stats_kernel']['frac'],3), 'K1b', round(k['hbar_reduce_kernel']['ms_per_launch'],4), 'K2', round(k['select_kernels']['ms_per_launch'],4), 'step', round(j['ms_per_step'],3))"
  done
done
