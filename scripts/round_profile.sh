# full GPU round: tests, bench (all legs), ncu launch list + full capture of one step's sampler launches
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(count|write)|k_total|DeviceScanKernel<detail::policy_hub<long, long" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(count|write)_" -s 8 -c 8 -o gpurun_out/prof python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
