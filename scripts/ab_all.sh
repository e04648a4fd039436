for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2311_17410_b200/libgfb200.so; else lib=$PWD/scripts/lib_$v.so; fi
  GF_LIB_PATH=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-fetch 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,2), d['ms_per_step'], {k.split('[')[1]:v['ms'] for k,v in d['kernels'].items()})"
done
