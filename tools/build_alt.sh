#!/bin/bash
# Build librsr_b200.so from another commit's csrc into build/alt/<name>/ (A/B kernel builds):
#   tools/build_alt.sh <commit> <name>
set -e
c=$1; name=$2; d=build/alt/$name
rm -rf $d; mkdir -p $d/src/paper_2411_06360_b200/csrc $d/src/include
git archive $c paper_2411_06360_b200/csrc include | tar -x -C $d/src
(cd $d/src && for f in paper_2411_06360_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -c $f -o ${f%.cu}.o & done; wait)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/librsr_b200.so $d/src/paper_2411_06360_b200/csrc/*.o -lcudart
echo built $d/librsr_b200.so
