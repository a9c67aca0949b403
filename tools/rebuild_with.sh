#!/bin/bash
# Rebuild ONE source of libsvgear.so with extra nvcc flags and relink (experiments on the GPU box):
#   tools/rebuild_with.sh seed.cu "-DSVG_SEED_GREEDY=0"
cd "$(dirname "$0")/.."
B=paper_2603_08982_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC $2 \
  -c -o $B/${1%.cu}.o paper_2603_08982_b200/csrc/$1 2>/dev/null || exit 1
nvcc -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -o paper_2603_08982_b200/libsvgear.so $B/*.o -lcuda || exit 1
