# A/B: library variants (GF_LIB_PATH) x write lanes
run() { GF_LIB_PATH=$1 GF_WRITE_LANES=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$3', d['value'], d['ms_per_step'], {k.split(')')[-1]:v['ms'] for k,v in d['kernels'].items() if 'fast' in k})"; }
run $PWD/paper_2311_17410_b200/libgfb200.so 16 keep16
run $PWD/scripts/libgfb200_nokeep.so 16 nokeep16
run $PWD/scripts/libgfb200_nokeep.so 8 nokeep8
