# round-2 batch x: overlap row-store alignment fix -- pairing tests incl. odd ranges, full sanitizer pass
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "pairing or qrange or range or shard" 2>&1 | tail -3 > gpurun_out/gpu_tests_x.log
for tool in memcheck racecheck synccheck initcheck; do
  q=--quick; [ $tool = memcheck ] && q=
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py $q > gpurun_out/sanitize_r02x_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_r02x_$tool.log
done
