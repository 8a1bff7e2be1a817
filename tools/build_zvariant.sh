#!/bin/bash
# Development: build paper_2003_04776_b200/libzz_<name>.so with zz_complex.cu compiled under the
# given -D flags (the other objects from the last in-tree build).
#   tools/build_zvariant.sh name "-DZZ_ZBK=8 -DZZ_ZSTAGES=5"
cd "$(dirname "$0")/../paper_2003_04776_b200"
v=$1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $2 \
     -c -o /tmp/zc_$v.o csrc/zz_complex.cu 2>&1 | grep -A2 -E "k_zdiag|k_zupdate" | grep -E "Used|spill" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libzz_$v.so $(ls build/*.o | grep -v zz_complex) /tmp/zc_$v.o \
     -L/usr/local/cuda/lib64 -ldl -Xlinker -rpath -Xlinker /usr/local/cuda/lib64 || exit 1
