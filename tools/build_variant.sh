#!/bin/bash
# Development: build paper_2003_04776_b200/libzz_<V>.so with zz_diag3.cu compiled under -DZZ_VARIANT_<V>
# (the other objects from the last in-tree build).
cd "$(dirname "$0")/../paper_2003_04776_b200"
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DZZ_VARIANT_$v \
       -c -o /tmp/d3_$v.o csrc/zz_diag3.cu || exit 1
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libzz_$v.so $(ls build/*.o | grep -v zz_diag3) /tmp/d3_$v.o \
       -L/usr/local/cuda/lib64 -ldl -Xlinker -rpath -Xlinker /usr/local/cuda/lib64 || exit 1
done
