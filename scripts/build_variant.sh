#!/bin/bash
# build an A/B variant of libst.so: recompile ONE source with extra flags, link with the other objects
# usage: build_variant.sh SRC.cu OUT.so "-DFLAG=..."
set -e
cd "$(dirname "$0")/../paper_2508_09589_b200"
src=$1; out=$2; extra=$3
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I../include -Icsrc $extra -c csrc/$src -o /tmp/variant_${src%.cu}.o
objs=$(ls build/*.o | grep -v "build/${src%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs /tmp/variant_${src%.cu}.o -lcudart
echo built $out
