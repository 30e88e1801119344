L=$PWD/paper_2602_01077_b200/lib
for lib in libpisa_b200_spec0.so libpisa_b200_spec1k3.so libpisa_b200.so; do
  for cfg in "1 33000 64 clustered 1 0.75" "1 33000 128 gaussian 0 0.875" "1 16424 128 gaussian 0 0.875"; do
    PISA_B200_LIB=$L/$lib timeout 60 python tools/repro_d64.py $cfg > /tmp/o.txt 2>&1 && echo "$lib $cfg ok" >> gpurun_out/repro_x.log || echo "$lib $cfg FAIL" >> gpurun_out/repro_x.log
  done
done
