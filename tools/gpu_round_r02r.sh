# round-2 batch r: bench with NVML clock sampling (short image steps too) + K/V stream field
timeout 300 python bench.py --workload flux --no-cpu --no-e2e > gpurun_out/r_flux.json 2> gpurun_out/r_flux.err
timeout 300 python bench.py --steps 3 --no-cpu --no-e2e --no-dense > gpurun_out/r_wan.json 2> gpurun_out/r_wan.err
