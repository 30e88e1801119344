#!/bin/bash
# A/B of the both-use exp2 split (PISA_POLY_BOTH) on clustered and gaussian
# routing: bash tools/ab_poly.sh b00 b11 ...  (libraries from tools/buildvar.sh)
cd /root/repo
for d in clustered gaussian; do
  for r in 1 2; do
    for n in "$@"; do
      L=$PWD/paper_2602_01077_b200/lib/libpisa_b200_$n.so
      PISA_B200_LIB=$L timeout 300 python bench.py --data $d --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$n', '$d', round(j['ms_per_step'],3), 'fused', round(k['fused_attn_kernel']['ms_per_launch'],3), 'exec_tflops', round(j['roofline']['executed_tflops']), 'U/k', round(j['roofline']['union_over_k'],3), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
    done
  done
done
for n in "$@"; do
  PISA_B200_LIB=$PWD/paper_2602_01077_b200/lib/libpisa_b200_$n.so timeout 600 python -m pytest tests/test_gpu.py -q -m gpu -k "fused_matches or randomized or golden" 2>&1 | tail -1 | sed "s/^/$n parity: /"
done
