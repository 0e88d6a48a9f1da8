#!/bin/bash
# Build libdma with extra -D flags into build_<name>/libdma.so:  build_variant.sh name "-DFOO=1 ..."
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_$name
for src in paper_2604_03950_b200/csrc/*.cu; do
  f=$(basename $src .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -Iinclude $* -c $src -o build_$name/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_$name/libdma.so build_$name/*.o
