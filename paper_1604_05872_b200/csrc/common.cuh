// common.cuh -- device helpers shared by the femgpu element kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace femgpu {

// SM count of the current device (B200: 148 = 2 dies x 74), queried once per
// device: persistent grids are sized from it, not from a constant.
inline int num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;  // benign race: every writer stores the same value
  }
  return cache[dev];
}

// ---------------------------------------------------------------------------
// Affine geometry: the level-1 preheader of every femopt IR
// (paper_1604_05872_b200/ir.py geometry_statements).
//   J_ab = x_{b+1,a} - x_{0,a},  K = J^{-1} = adj(J)/det,  adet = |det J|.
// x points at the cell's 12 coordinates [4][3].
// ---------------------------------------------------------------------------
struct Geo {
  double K[3][3];
  double adet;
};

__device__ __forceinline__ Geo cell_geometry(const double* x) {
  double J[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) J[a][b] = x[(b + 1) * 3 + a] - x[a];
  double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
  double r = 1.0 / det;
  Geo g;
  g.adet = fabs(det);
  // K_ab = C_ba / det
  g.K[0][0] = c00 * r;
  g.K[1][0] = c01 * r;
  g.K[2][0] = c02 * r;
  g.K[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * r;
  g.K[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * r;
  g.K[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * r;
  g.K[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * r;
  g.K[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * r;
  g.K[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * r;
  return g;
}

// ---------------------------------------------------------------------------
// FP64 tensor core: mma.sync m16n8k8 (executes as 4x DMMA.8x8x4 on sm_100a;
// measured 37.0 TFLOP/s, profiles/fp64_peak_r01.txt).  Fragment layouts
// (lane = 4*g + t):
//   A (16x8, row):  a[v] = A[g + 8*(v&1)][t + 4*(v>>1)]
//   B (8x8,  col):  b[v] = B[t + 4*v][g]
//   C (16x8):       c[v] = C[g + 8*(v>>1)][2*t + (v&1)]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma16x8x8(double (&c)[4], const double (&a)[4],
                                           const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// ---------------------------------------------------------------------------
// mbarrier + 1D TMA bulk copy (cp.async.bulk, SASS UBLKCP).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16B aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 cache policy for streaming writes (createpolicy; used as a .L2::cache_hint operand).
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
// Shared -> global bulk copy (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
// Shared -> global bulk reduction (A += staged), bulk-group completion.
__device__ __forceinline__ void bulk_s2g_add(double* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

// read-once 16-byte load of index data (no L1 allocation)
__device__ __forceinline__ longlong2 ldg_stream_idx(const longlong2* p) {
  longlong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s64 {%0,%1}, [%2];\n"
               : "=l"(v.x), "=l"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1,%2};\n" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

}  // namespace femgpu
