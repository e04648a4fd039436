# ncu evidence for the feature-fetch row copy (k_fetch_gather) inside the bench's fetch block, and the
# ingest launch list (per-kernel durations of 100K-edge batches, graph replay off so kernels are separable).
# Run from the repo root under gpurun.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fetch_gather" -s 8 -c 2 \
  -o gpurun_out/prof_fetch python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
GF_INGEST_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ingest_launches.csv python scripts/ingest_profile.py 2000000 100000 > /dev/null 2>&1
ls gpurun_out
