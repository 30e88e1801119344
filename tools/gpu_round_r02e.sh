# round-2 batch e: L2 / fabric metrics of the fused kernel (previous design) on
# gaussian vs clustered routing: is it bound by L2 -> SM delivery or L2 slice hot-spots?
set -x
L=$PWD/paper_2602_01077_b200/lib
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.max,lts__t_sectors.avg,lts__t_sectors_srcunit_tex.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__d_sectors_fill_sysmem.sum,lts__t_requests_srcunit_tex.sum,lts__average_t_sector_hit_rate_realtime.pct
for d in gaussian clustered; do
  PISA_B200_LIB=$L/libpisa_b200_k3old.so timeout 600 ncu --metrics $M --clock-control none -k regex:fused_attn -s 3 -c 1 --csv python bench.py --data $d --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/l2_$d.csv 2> gpurun_out/l2_$d.err
done
ncu --query-metrics 2>/dev/null | grep -i -E "^lts__|ltcfabric|nvlrx|xbar" | head -60 > gpurun_out/l2_metric_names.txt
