#!/bin/bash
# recent-policy A/B over library variants (scripts/build_variant.sh): sampler-only bench per variant
scripts/quick_bench.sh base
GF_NO_MEMO=1 scripts/quick_bench.sh nomemo
for v in "$@"; do GF_LIB_PATH=scripts/lib_$v.so scripts/quick_bench.sh $v; done
