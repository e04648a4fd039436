#!/bin/bash
# A/B the mag8 bench over library variants: scripts/ab_mag.sh name1 name2 ... ("base" = in-tree library)
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2311_17410_b200/libgfb200.so; else lib=$PWD/scripts/lib_$v.so; fi
  GF_LIB_PATH=$lib timeout 600 python bench.py --config mag8 --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,2), 'G/s', d['ms_per_step'], 'ms', {k:v['ms'] for k,v in d['kernels'].items()})" || echo "$v failed"
done
