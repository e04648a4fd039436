#!/bin/bash
# Round-2 evidence run (repo root, under gpurun): every bench configuration, the ncu sampler captures
# and the ingest profile, into gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_gdelt.json 2> gpurun_out/final_gdelt.err
for c in mag8 reddit wiki; do
  timeout 900 python bench.py --config $c > gpurun_out/final_$c.json 2> gpurun_out/final_$c.err
done
timeout 900 python bench.py --deleted --no-cpu > gpurun_out/final_gdelt_deleted.json 2> gpurun_out/final_gdelt_deleted.err
timeout 600 python bench.py --impl reference > gpurun_out/final_reference.json 2> gpurun_out/final_reference.err
bash scripts/ncu_sampler.sh > /dev/null 2>&1
timeout 300 python scripts/ingest_profile.py 20000000 100000 > gpurun_out/final_ingest_gdelt.txt 2>&1
timeout 300 python scripts/ingest_profile.py 80000000 10000000 15250000 120 > gpurun_out/final_ingest_mag8.txt 2>&1
ls -la gpurun_out | tail -20
