#!/bin/bash
# A/B of the fused kernel: old library vs current (persistent / one CTA per tile)
cd /root/repo
run() {  # label lib persistent workload steps
  PISA_B200_LIB=$2 PISA_B200_PERSISTENT=$3 timeout 300 python bench.py --workload $4 --steps $5 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$1 $4', round(j['ms_per_step'],4), 'fused', round(j['kernels']['fused_attn_kernel']['ms_per_launch'],4), j['clocks']['sm_mhz'])"
}
OLD=$PWD/paper_2602_01077_b200/lib/libpisa_b200_old.so
NEW=$PWD/paper_2602_01077_b200/lib/libpisa_b200.so
for r in 1 2; do
  for w in "wan14b 10" "flux 50" "wan13b 20"; do
    set -- $w
    run old $OLD 1 $1 $2; run pers $NEW 1 $1 $2; run tile $NEW 0 $1 $2
  done
done
