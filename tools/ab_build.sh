#!/bin/bash
# Build an A/B variant of the library with extra -D flags on one source file:
#   bash tools/ab_build.sh <name> <source.cu> -DFOO=1 ...   ->  build/ab/lib<name>.so
set -e
name=$1; src=$2; shift 2
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude"
mkdir -p build/ab/$name
base=$(basename $src .cu)
$NV $FL "$@" -c -o build/ab/$name/$base.o paper_2208_06290_b200/csrc/$src
objs=""
for o in build/obj/*.o; do
  if [ "$(basename $o)" = "$base.o" ]; then objs="$objs build/ab/$name/$base.o"; else objs="$objs $o"; fi
done
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/ab/lib$name.so $objs
echo built build/ab/lib$name.so
