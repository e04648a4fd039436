for g in 32 64 128; do
  GF_L2_FETCH_GRANULARITY=$g timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e > gpurun_out/l2_$g.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/l2_$g.log').read().strip().splitlines()[-1]); print($g, d['value'], d['ms_per_step'], json.dumps(d['kernels']))"
done
