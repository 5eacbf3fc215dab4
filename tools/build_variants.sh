#!/bin/bash
# Build libjdob variants with different -D flags into tools/ (optimisation experiments).
# usage: tools/build_variants.sh NAME "FLAGS" [NAME "FLAGS" ...]
set -e
cd "$(dirname "$0")/../paper_2504_14611_b200"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=/tmp/var_$name; mkdir -p $d
  for f in aggregates solve eval stats bruteforce grouping solve_large gen api; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden $flags -c csrc/$f.cu -o $d/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../tools/libjdob_$name.so $d/*.o -cudart static
done
