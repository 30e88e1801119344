cd /root/repo
for d in gaussian clustered; do for L in c8 c16 c16w96; do
PISA_B200_LIB=$PWD/paper_2602_01077_b200/lib/libpisa_b200_$L.so timeout 300 python bench.py --data $d --steps 10 --warmup 3 --no-cpu --no-e2e --no-dense 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$L $d', round(j['ms_per_step'],3), 'fused', round(k['fused_attn_kernel']['ms_per_launch'],3), 'pair', round(k['pairing_kernels']['ms_per_launch'],3), 'U/k', round(j['roofline']['union_over_k'],4), j['clocks']['sm_mhz'])"
done; done
