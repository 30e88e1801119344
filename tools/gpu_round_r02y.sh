PISA_B200_LIB=$PWD/paper_2602_01077_b200/lib/libpisa_b200_trace.so timeout 120 python tools/trace_hang.py 1 16424 128 gaussian 0 0.875 128 > gpurun_out/trace_hang.txt 2>&1
