#!/bin/sh
# Development build of libfemgpu with the Burgers pipeline trace (-DBZ_TRACE -DET_TRACE).
set -e
cd "$(dirname "$0")/../paper_1604_05872_b200/csrc"
mkdir -p build/trace
for f in capi helmholtz helm_quad pair elasticity burgers global vector gemm_f64 svk_mma burgers_quad; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -DBZ_TRACE -DET_TRACE -c $f.cu -o build/trace/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/libfemgpu_trace.so \
  build/trace/capi.o build/trace/helmholtz.o build/trace/helm_quad.o build/trace/pair.o build/trace/elasticity.o build/trace/burgers.o build/trace/global.o build/trace/vector.o build/trace/gemm_f64.o build/trace/svk_mma.o build/trace/burgers_quad.o -lcudart -ldl
