#!/bin/bash
# Build one libcohere_b200 variant with one CUDA source recompiled with extra -D flags into
# paper_1910_11110_b200/lib/variants/TAG.so (select with COH_B200_LIB; scripts/te_variants.py,
# scripts/runs_variants.py).
# usage: scripts/build_variant.sh SRC.cu TAG [-DNAME=VALUE ...]
set -e
cd "$(dirname "$0")/../paper_1910_11110_b200"
src=$1; tag=$2; shift 2
base=$(basename "$src" .cu)
make -C csrc -j8 >/dev/null
mkdir -p lib/variants build/variants
OBJS=$(ls build/*.o | grep -v "/$base.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I../include -Icsrc -Xptxas -v "$@" -c csrc/$src -o build/variants/${base}_$tag.o 2> build/variants/${base}_$tag.ptxas.txt
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o lib/variants/$tag.so build/variants/${base}_$tag.o $OBJS -lpthread -ldl -lrt
echo "$tag: $(grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' build/variants/${base}_$tag.ptxas.txt | sort | uniq -c | tr '\n' ' ')"
