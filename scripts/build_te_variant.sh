#!/bin/bash
# Build one libcohere_b200 variant with extra -D flags for trace_eval.cu into
# paper_1910_11110_b200/lib/variants/TAG.so (select with COH_B200_LIB; scripts/te_variants.py).
# usage: scripts/build_te_variant.sh TAG [-DNAME=VALUE ...]
set -e
cd "$(dirname "$0")/../paper_1910_11110_b200"
tag=$1; shift
make -C csrc -j8 >/dev/null
mkdir -p lib/variants build/variants
OBJS=$(ls build/*.o | grep -v trace_eval.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I../include -Icsrc -Xptxas -v "$@" -c csrc/trace_eval.cu -o build/variants/te_$tag.o 2> build/variants/te_$tag.ptxas.txt
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o lib/variants/$tag.so build/variants/te_$tag.o $OBJS -lpthread -ldl -lrt
for k in 12 20; do
  echo "$tag <$k>: $(grep -A2 "k_trace_evalILi${k}E" build/variants/te_$tag.ptxas.txt | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ')"
done
