#!/bin/bash
# A/B the post-deletion sampler (bench.py --deleted) over library variants: scripts/ab_deleted.sh base name ...
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2311_17410_b200/libgfb200.so; else lib=$PWD/scripts/lib_$v.so; fi
  GF_LIB_PATH=$lib timeout 600 python bench.py --deleted --steps 5 --warmup 3 --no-cpu --no-e2e --no-fetch 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,2), 'G/s', d['ms_per_step'], 'ms', {k:v['ms'] for k,v in d['kernels'].items()})" || echo "$v failed"
done
