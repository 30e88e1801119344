# round-2 batch l: K1 diagnostics -- column warps skipped (k1d1) / H partial store skipped (k1d2)
set -x
L=paper_2602_01077_b200/lib
sel() { python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$1', round(j['ms_per_step'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()}, j['clocks']['sm_mhz'])"; }
for r in 1 2; do
  for v in "" k1d1 k1d2; do
    lib=$L/libpisa_b200${v:+_$v}.so
    for w in flux wan14b; do
      PISA_B200_LIB=$lib timeout 300 python bench.py --workload $w --steps 5 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | sel "$w ${v:-base}" >> gpurun_out/ab_k1_l.log 2>&1
    done
  done
done
