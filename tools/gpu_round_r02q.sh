# round-2 batch q: image-size breakdowns (plain / covariance router), current library
for w in flux sd35; do for r in plain covariance; do
  timeout 300 python bench.py --workload $w --router $r --no-cpu --no-e2e > gpurun_out/img_${w}_${r}.json 2> gpurun_out/img_${w}_${r}.err
done; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_flux_cov.csv python bench.py --workload flux --router covariance --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense > /dev/null 2>&1
