#!/bin/bash
# build an A/B variant of libgfb200.so: scripts/build_variant.sh NAME -DFLAG=... ; load with GF_LIB_PATH=scripts/lib_NAME.so
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2311_17410_b200/csrc"
out=/tmp/variant_$name; mkdir -p $out
for f in gf_util gf_graph gf_sample gf_cache gf_offload gf_part; do
  nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -gencode arch=compute_100a,code=sm_100a \
       --expt-relaxed-constexpr "$@" -c $f.cu -o $out/$f.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../../scripts/lib_$name.so $out/*.o -lcudart_static -lrt -ldl -lpthread
echo built scripts/lib_$name.so
