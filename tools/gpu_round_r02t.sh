# round-2 batch t: full GPU suite on the new default (single-pass softmax, 2 K stages); the fused-select test alone, verbose
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/gpu_tests_t.log
for cfg in "1 33000 64 clustered 1 0.75" "1 16424 128 gaussian 0 0.875"; do timeout 60 python tools/repro_d64.py $cfg >> gpurun_out/gpu_tests_t.log 2>&1; done
PISA_B200_FUSED_SELECT=1 timeout 300 python -m pytest tests/test_gpu.py -m gpu -q -x -k "fused_select" 2>&1 | tail -40 > gpurun_out/gpu_tests_t_fsel.log
