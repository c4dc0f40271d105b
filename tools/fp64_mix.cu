// fp64_mix.cu -- do DMMA (mma.sync f64) and DFMA share one FP64 pipe on sm_100a?
// Half the warps of each CTA run m16n8k4 chains, half run DFMA chains; compare the
// combined rate with each alone.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(double* out, int iters, int mode) {  // mode 0 both, 1 dmma only, 2 dfma only
  const int warp = threadIdx.x >> 5;
  const bool mma_warp = ((warp >> 2) & 1) == 0;  // both kinds on every SMSP
  double s = 0;
  if (mma_warp && mode != 2) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1 - a0;
    double c[4][4] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a0), "d"(a1), "d"(b));
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][3];
  } else if (!mma_warp && mode != 1) {
    double acc[8];
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x + k;
    for (int it = 0; it < 4 * iters; ++it)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fma(acc[k], 0.999, 1e-3);
    for (int k = 0; k < 8; ++k) s += acc[k];
  }
  if (s == 1234.5) out[0] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, tpb = 512, grid = p.multiProcessorCount;
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<grid, tpb>>>(out, iters, mode);
    cudaEventRecord(e0);
    mix<<<grid, tpb>>>(out, iters, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // per CTA: 8 mma warps x 4 chains x iters m16n8k4 (1024 flop); 8 dfma warps x 32 lanes x 8 x 4 iters x 2
    double fm = 8.0 * 4 * iters * 1024 * grid, ff = 8.0 * 32 * 8 * 4 * iters * 2 * grid;
    printf("mode %s: %.3f ms  dmma %.1f TF  dfma %.1f TF\n", mode == 0 ? "both " : mode == 1 ? "dmma " : "dfma ",
           ms, mode != 2 ? fm / ms / 1e9 : 0.0, mode != 1 ? ff / ms / 1e9 : 0.0);
  }
  return 0;
}
