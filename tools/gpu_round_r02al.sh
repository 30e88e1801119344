L=$PWD/paper_2602_01077_b200/lib
for d in clustered gaussian; do
  PISA_B200_LIB=$L/libpisa_b200_trace.so timeout 300 python tools/trace_timeline.py 40 $d > gpurun_out/trace_cur_$d.txt 2>&1
done
