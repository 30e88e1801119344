#!/bin/bash
# K1c phase clocks (libs c1..c5) and baseline vs variant timing / parity: k1c_ab.sh [variant ...]
cd /root/repo
L=$PWD/paper_2602_01077_b200/lib
for i in 1 2 3 4 5; do PISA_B200_LIB=$L/libpisa_b200_c$i.so timeout 300 python tools/k1c_probe.py clocks c$i; done
echo "(c1 Lanczos loop, c2 ritz, c3 preparation, c4 whole CTA, c5 K/V TMA wait)"
for r in 1 2; do
  for n in base "$@"; do
    lib=$L/libpisa_b200.so; [ $n != base ] && lib=$L/libpisa_b200_$n.so
    PISA_B200_LIB=$lib timeout 300 python tools/k1c_probe.py time $n
    for w in wan14b flux; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --router covariance --no-cpu --no-e2e --no-dense --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$n', '$w', round(j['ms_per_step'],4), 'k1c', round(j['kernels']['block_norms_kernel']['ms_per_launch'],4))"
    done
  done
done
for n in "$@"; do python tools/k1c_probe.py compare $n base; done
