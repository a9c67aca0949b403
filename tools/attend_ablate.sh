#!/bin/bash
# Ablations of the attention kernel (timing only): rebuilds attend_tc.o with -DSVG_ABL=<bits> on the GPU
# box, relinks libsvgear.so and times the kernel alone.  Bits: 1 no softmax arithmetic, 2 never redo,
# 4 no QK^T MMAs, 8 no P.V MMAs.  Usage: tools/attend_ablate.sh "0 3 14 6 10 7 11"
cd "$(dirname "$0")/.."
B=paper_2603_08982_b200/build
for abl in $1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -DSVG_ABL=$abl $EXTRA \
    -c -o $B/attend_tc.o paper_2603_08982_b200/csrc/attend_tc.cu || exit 1
  nvcc -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -o paper_2603_08982_b200/libsvgear.so $B/*.o -lcuda || exit 1
  echo "ABL=$abl $EXTRA: $(HEADS=${HEADS:-8} timeout 300 python tools/attend_time.py 2>&1 | tail -1)"
done
