// hbm_bw.cu -- streaming read / write / copy bandwidth on this B200 (context for
// the write-dominated element-matrix kernels; MEASURED_PEAKS.json has copy only).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void wr(double2* __restrict__ b, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v2.f64 [%0], {%1,%1};" ::"l"(b + i), "d"(v) : "memory");
}
__global__ void rd(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a + i));
    s += v.x + v.y;
  }
  if (s == 1.2345) out[0] = s;
}
__global__ void cp(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
int main() {
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer
  double2 *a, *b;
  double* o;
  cudaMalloc(&a, n * 16);
  cudaMalloc(&b, n * 16);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, n * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {4, 8, 16}) {
    int grid = 148 * bps;
    float best_w = 1e9, best_r = 1e9, best_c = 1e9, ms;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); wr<<<grid, 512>>>(b, n, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best_w) best_w = ms;
      cudaEventRecord(e0); rd<<<grid, 512>>>(a, n, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best_r) best_r = ms;
      cudaEventRecord(e0); cp<<<grid, 512>>>(a, b, n / 2); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best_c) best_c = ms;
    }
    printf("blocks/SM %2d: write %.0f GB/s  read %.0f GB/s  copy(r+w) %.0f GB/s\n", bps,
           n * 16 / best_w / 1e6, n * 16 / best_r / 1e6, n * 16 / best_c / 1e6);
  }
  return 0;
}
