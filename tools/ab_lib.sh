#!/bin/bash
# A/B two libraries on the bench (fused ms, pairing ms, union/k): ab_lib.sh libA libB [data ...]
cd /root/repo
A=$1; B=$2; shift 2
for d in "${@:-gaussian}"; do
  for r in 1 2; do
    for L in $A $B; do
      PISA_B200_LIB=$L timeout 300 python bench.py --data $d --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$(basename $L)', '$d', round(j['ms_per_step'],3), 'fused', round(k['fused_attn_kernel']['ms_per_launch'],3), 'pair', round(k.get('pairing_kernels',{}).get('ms_per_launch',0),3), 'U/k', round(j['roofline']['union_over_k'],3), j['clocks']['sm_mhz'])"
    done
  done
done
