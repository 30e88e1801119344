#!/bin/bash
# A/B the routing kernels (score + top-k) across libraries: ab_select.sh name ... (base = libpisa_b200.so)
cd /root/repo
L=$PWD/paper_2602_01077_b200/lib
for r in 1 2; do
  for n in "$@"; do
    lib=$L/libpisa_b200.so; [ $n != base ] && lib=$L/libpisa_b200_$n.so
    for w in wan14b flux; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --no-cpu --no-e2e --no-dense --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$n', '$w', round(j['ms_per_step'],4), 'select', round(k['select_kernels']['ms_per_launch'],4), 'stats', round(k['block_stats_kernel']['ms_per_launch'],4))"
    done
  done
done
