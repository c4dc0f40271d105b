// dmma_shapes.cu -- FP64 mma.sync throughput/latency per shape vs independent
// chains and warps per SM sub-partition (development aid for the element kernels).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_shapes dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = 1.0 + a0, b = 1.0 - threadIdx.x * 1e-4;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int i = 0; i < 4; ++i) c[k][i] = k + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int i = 0; i < 4; ++i) s += c[k][i];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void k8(double* out, int iters) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int i = 0; i < 4; ++i) c[k][i] = k + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) for (int i = 0; i < 4; ++i) s += c[k][i];
  if (s == 12345.678) out[0] = s;
}

template <class F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

template <int CH>
void run(int sms, double* out) {
  const int iters = 2048;
  for (int wps : {1, 2, 4}) {  // warps per SMSP (1 CTA per SM, 4*wps warps)
    int tpb = 128 * wps;
    float ms = time_it([&] { k4<CH><<<sms, tpb>>>(out, iters); });
    double fl = 2.0 * 16 * 8 * 4 * CH * iters * (double)sms * (tpb / 32);
    double cyc = ms * 1e-3 * 1.965e9;
    printf("m16n8k4 chains=%d warps/SMSP=%d: %6.2f TFLOP/s  cycles/mma/warp %.1f\n", CH, wps,
           fl / ms / 1e9, cyc / (CH * (double)iters));
    ms = time_it([&] { k8<CH><<<sms, tpb>>>(out, iters); });
    fl = 2.0 * 16 * 8 * 8 * CH * iters * (double)sms * (tpb / 32);
    cyc = ms * 1e-3 * 1.965e9;
    printf("m16n8k8 chains=%d warps/SMSP=%d: %6.2f TFLOP/s  cycles/mma/warp %.1f\n", CH, wps,
           fl / ms / 1e9, cyc / (CH * (double)iters));
  }
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 8);
  run<1>(p.multiProcessorCount, out);
  run<2>(p.multiProcessorCount, out);
  run<3>(p.multiProcessorCount, out);
  run<4>(p.multiProcessorCount, out);
  run<8>(p.multiProcessorCount, out);
  return 0;
}
