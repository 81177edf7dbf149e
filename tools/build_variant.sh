#!/bin/bash
# Build the current csrc with extra nvcc defines into build/alt/<name>/librsr_b200.so (A/B of compile-time knobs):
#   tools/build_variant.sh <name> -DRSR_KA=1 ...
name=$1; shift
d=build/alt/$name; mkdir -p $d; rm -f $d/*.o
for f in paper_2411_06360_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o $d/$(basename ${f%.cu}).o 2>/dev/null &
done; wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xlinker -soname=librsr_b200.so -o $d/librsr_b200.so $d/*.o build/obj/*.cpp.o -lcudart && echo $d/librsr_b200.so
