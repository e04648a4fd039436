# ncu evidence for one sampling step: launch list (all step kernels) + full capture of the 4 fused sampler launches
# (recent/uniform x hop 0/1) of the timed step.  Run from the repo root under gpurun.
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sample_fused|k_count|k_write|k_total|DeviceScanKernel" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sample_fused" -s 4 -c 4 -o gpurun_out/prof python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
