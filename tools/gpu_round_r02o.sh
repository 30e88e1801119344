# round-2 batch o: L2 fabric (die-to-die) metrics of the fused kernel
ncu --query-metrics 2>/dev/null | grep -i -E "fabric|lts__t_sectors_srcnode|lts__t_sectors_srcunit|lts__t_requests_srcnode|gpc__|remote" > gpurun_out/fabric_metric_names.txt
M=$(grep -o -E "^lts__t_sectors_srcunit_ltcfabric[a-z_]*|^lts__ltcfabric[a-z_0-9]*|^lts__t_sectors_srcnode_[a-z_]*" gpurun_out/fabric_metric_names.txt | sort -u | sed 's/$/.sum/' | tr '\n' ',' | sed 's/,$//')
echo "$M" > gpurun_out/fabric_metrics_used.txt
L=$PWD/paper_2602_01077_b200/lib
PISA_B200_LIB=$L/libpisa_b200_k3old.so timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sectors.sum,$M --clock-control none -k regex:fused_attn -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-dense > gpurun_out/fabric_gaussian.csv 2> gpurun_out/fabric_gaussian.err
