#!/bin/bash
# A/B ingest throughput over library variants: scripts/ab_ingest.sh name1 name2 ... ("base" = in-tree library)
for v in "$@"; do
  if [ "$v" = base ]; then lib=$PWD/paper_2311_17410_b200/libgfb200.so; else lib=$PWD/scripts/lib_$v.so; fi
  echo -n "$v "; GF_LIB_PATH=$lib timeout 200 python scripts/ingest_profile.py 20000000 100000 2>&1 | grep unprofiled
done
