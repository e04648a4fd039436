# ncu evidence for one sampling step: launch list (all step kernels) + full capture of the 8 sampler launches
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_count_lane|k_write_coop|k_total|DeviceScanKernel" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_count_lane|k_write_coop" -s 8 -c 8 -o gpurun_out/prof python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
