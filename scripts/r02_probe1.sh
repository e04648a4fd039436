set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
GF_INGEST_TIMING=1 timeout 300 python scripts/ingest_profile.py 20000000 100000 > gpurun_out/ing_prof.txt 2>&1
GF_INGEST_NO_GRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 400 --csv --log-file gpurun_out/ing_launches.csv python scripts/ingest_profile.py 4000000 100000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sample_fused" -s 2 -c 2 -o gpurun_out/prof_mag python bench.py --config mag8 --steps 1 --warmup 1 --no-cpu --no-e2e --no-fetch > gpurun_out/mag_ncu.log 2>&1
ls -la gpurun_out
