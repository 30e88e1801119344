#!/bin/bash
# K1c A/B on one box: k1c_var.sh "clock-libs ..." "timed-libs ..." (names as built by buildvar.sh; base = libpisa_b200.so)
cd /root/repo
L=$PWD/paper_2602_01077_b200/lib
for n in $1; do PISA_B200_LIB=$L/libpisa_b200_$n.so timeout 300 python tools/k1c_probe.py clocks $n 2>&1 | grep -v Warn; done
for r in 1 2; do
  for n in $2; do
    lib=$L/libpisa_b200.so; [ $n != base ] && lib=$L/libpisa_b200_$n.so
    for w in wan14b flux; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --router covariance --no-cpu --no-e2e --no-dense --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$n', '$w', round(j['ms_per_step'],4), 'k1c', round(j['kernels']['block_norms_kernel']['ms_per_launch'],4))"
    done
  done
done
