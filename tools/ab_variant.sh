#!/bin/bash
# Build an A/B variant of libgsrcuda.so whose fast.cu comes from a file:
#   bash tools/ab_variant.sh <fast.cu> <name>   → scratch/libgsrcuda_<name>.so
# (every other object is the in-tree build; load it with GSRC_LIB=...)
set -e
SRC=$1; NAME=$2
O=paper_2603_27156_b200/csrc/_obj
T=paper_2603_27156_b200/csrc/_ab_fast_$NAME.cu; cp "$SRC" $T
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -c $T -o scratch/fast_$NAME.o
rm -f $T
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scratch/libgsrcuda_$NAME.so $O/kernels.o $O/tile_w32.o $O/tile_w64.o $O/tile_w128.o scratch/fast_$NAME.o $O/capi.o -Xcompiler -fPIC -ldl
echo scratch/libgsrcuda_$NAME.so
