for p in 0 64 96; do
  GF_L2_PERSIST=$p timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$p', d['value'], d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items() if 'count' in k})"
done
