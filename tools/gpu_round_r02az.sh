# round-2 batch az: compute-sanitizer over every kernel of the current library
for t in memcheck racecheck synccheck initcheck; do
  q=""; [ $t != memcheck ] && q="--quick"
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize.py $q > gpurun_out/san_$t.log 2>&1
  echo "$t exit=$?" >> gpurun_out/san_summary.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|calls" gpurun_out/san_$t.log | tail -3 >> gpurun_out/san_summary.log
done
