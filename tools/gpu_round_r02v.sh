for d in 64 128; do for kind in gaussian clustered; do for fd in 0 1; do
  timeout 60 python tools/repro_d64.py 1 8192 $d $kind $fd 0.75 >> gpurun_out/repro_v.log 2>&1 || echo "FAIL 1 8192 $d $kind $fd" >> gpurun_out/repro_v.log
done; done; done
timeout 60 python tools/repro_d64.py 1 2048 64 clustered 0 0.75 >> gpurun_out/repro_v.log 2>&1 || echo "FAIL small" >> gpurun_out/repro_v.log
timeout 300 compute-sanitizer --tool memcheck python tools/repro_d64.py 1 2048 64 clustered 0 0.75 > gpurun_out/repro_v_san.log 2>&1
