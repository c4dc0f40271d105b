#!/bin/sh
# Build libfemgpu from the current csrc into tools/ab/<name>.so (A/B timing, development).
set -e
name=$1
cd "$(dirname "$0")/../paper_1604_05872_b200/csrc"
mkdir -p build/ab ../../tools/ab
for f in capi helmholtz helm_quad pair elasticity burgers global vector gemm_f64 svk_mma burgers_quad; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr $2 -c $f.cu -o build/ab/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/ab/$name.so \
  build/ab/capi.o build/ab/helmholtz.o build/ab/helm_quad.o build/ab/pair.o build/ab/elasticity.o build/ab/burgers.o build/ab/global.o build/ab/vector.o build/ab/gemm_f64.o build/ab/svk_mma.o build/ab/burgers_quad.o -lcudart -ldl
