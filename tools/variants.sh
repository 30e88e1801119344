#!/bin/bash
# A/B the fused kernel across library variants built by tools/buildvar.sh:
#   bash tools/variants.sh name1 name2 ...   (prints fused ms + parity per variant)
for n in "$@"; do
  export PISA_B200_LIB=$PWD/paper_2602_01077_b200/lib/libpisa_b200_$n.so
  timeout 300 python bench.py --no-e2e --no-cpu --no-dense --steps 10 > gpurun_out/var_$n.json 2>/dev/null
  ok=$(timeout 300 python tools/gpu_diag.py 2>&1 | grep -c FAIL)
  python -c "
import json; j=json.load(open('gpurun_out/var_$n.json')); print('$n', 'fused', round(j['kernels']['fused_attn_kernel']['ms_per_launch'],3), 'total', round(j['ms_per_step'],3), 'diag FAILs: $ok', j['clocks']['sm_mhz'])"
done
