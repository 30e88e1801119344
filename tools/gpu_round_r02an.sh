L=$PWD/paper_2602_01077_b200/lib
PISA_B200_LIB=$L/libpisa_b200_mw256tr.so timeout 300 python tools/trace_timeline.py 40 clustered > gpurun_out/trace_mw256_clustered.txt 2>&1
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_mw256.so clustered gaussian > gpurun_out/ab_k3_an.log 2>&1
