#!/bin/bash
# Build an A/B variant of libwagma_b200.so with extra -D defines: tools/build_variant.sh out.so -DFOO=1 ...
OUT=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 -shared \
  -I include "$@" -o "$OUT" -diag-suppress 1886,177 paper_2005_00124_b200/csrc/wagma_b200.cu paper_2005_00124_b200/csrc/topology.cpp
