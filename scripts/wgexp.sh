for wg in 16 8 4; do
  GF_WRITE_LANES=$wg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/wg_$wg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/wg_$wg.log').read().strip().splitlines()[-1])
print($wg, d['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items() if 'write' in k})"
done
