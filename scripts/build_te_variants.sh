#!/bin/bash
# Build libcohere_b200 variants with different trace_eval block sizes / occupancy
# targets into paper_1910_11110_b200/lib/variants/ (select one with COH_B200_LIB=...).
set -e
cd "$(dirname "$0")/../paper_1910_11110_b200"
make -C csrc -j8 >/dev/null
mkdir -p lib/variants build/variants
OBJS=$(ls build/*.o | grep -v trace_eval.o)
for v in "$@"; do  # v = NT:MINB_DOUBLE:MINB
  IFS=: read nt md ms <<< "$v"
  tag="nt${nt}_d${md}_s${ms}"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I../include -Icsrc -Xptxas -v -DCOH_TE_NT=$nt -DCOH_TE_MINB_DOUBLE=$md -DCOH_TE_MINB=$ms \
    -c csrc/trace_eval.cu -o build/variants/te_$tag.o 2> build/variants/te_$tag.ptxas.txt
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
    -o lib/variants/libcohere_b200_$tag.so build/variants/te_$tag.o $OBJS -lpthread -ldl -lrt
  echo "$tag: $(grep -A2 'k_trace_evalILi12E' build/variants/te_$tag.ptxas.txt | grep -o 'Used [0-9]* registers') (double)," \
       "$(grep -A2 'k_trace_evalILi4E' build/variants/te_$tag.ptxas.txt | grep -o 'Used [0-9]* registers\|[0-9]* bytes spill stores' | tr '\n' ' ') (single)"
done
