#!/bin/bash
# Build the -DDMA_PROFILE variant (per-phase softmax cycle counters) into build_prof/libdma_prof.so
cd "$(dirname "$0")/.."
mkdir -p build_prof
for f in capi_attn capi_quant selftest; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude -DDMA_PROFILE $EXTRA -c paper_2604_03950_b200/csrc/$f.cu -o build_prof/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_prof/libdma_prof.so build_prof/*.o
