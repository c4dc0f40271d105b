// global.cu -- the steps either side of the path:
// gather of per-cell inputs from global vectors before it, scatter-add of the
// element matrices into a global CSR matrix after it.
//
// The reference stops at the element matrix and reads pre-gathered
// per-cell tables (proj/tests/kernels.hpp:186-188); a FEM code around it
// performs these two steps.  Both are HBM/latency-bound integer-indexed
// streams, so they are written as such (no tensor cores): grid-stride over the
// output index space with coalesced stores (gather) and coalesced loads +
// FP64 atomics (scatter).  The CSR positions of a cell's n x n entries depend
// only on the mesh, so they are resolved once (binary search in the sorted
// row) and reused by every assembly -- the usual split between symbolic and
// numeric assembly.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

namespace {

__global__ void gather_kernel(long E, int ncoef, const double* __restrict__ V,
                              const int* __restrict__ cells, const double* __restrict__ coef,
                              const int* __restrict__ coef_idx, double* __restrict__ coords,
                              double* __restrict__ coeffs) {
  const long nx = E * 12, total = nx + E * (long)ncoef;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    if (t < nx) {  // coords[e][v][c] = V[cells[e][v]][c]
      const long e = t / 12;
      const int r = (int)(t - e * 12), v = r / 3, c = r - 3 * v;
      coords[t] = __ldg(&V[(long)__ldg(&cells[e * 4 + v]) * 3 + c]);
    } else {  // coeffs[e][s] = coef[coef_idx[e][s]]
      const long u = t - nx;
      coeffs[u] = __ldg(&coef[__ldg(&coef_idx[u])]);
    }
  }
}

// pos[e][j][k] = index of column dof[e][k] in row dof[e][j] (-1 if absent)
__global__ void csr_positions_kernel(long E, int n, const int* __restrict__ dof,
                                     const long* __restrict__ row_ptr,
                                     const int* __restrict__ col_idx, long* __restrict__ pos,
                                     int* __restrict__ missing) {
  const long rows = E * (long)n;
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < rows;
       t += (long)gridDim.x * blockDim.x) {
    const long e = t / n;
    const int r = __ldg(&dof[t]);
    const long b = __ldg(&row_ptr[r]), len = __ldg(&row_ptr[r + 1]) - b;
    const int* cols = col_idx + b;
    long* out = pos + t * n;
    for (int k = 0; k < n; ++k) {
      const int c = __ldg(&dof[e * n + k]);
      long lo = 0, hi = len;  // first column >= c
      while (lo < hi) {
        const long mid = (lo + hi) >> 1;
        if (__ldg(&cols[mid]) < c) lo = mid + 1; else hi = mid;
      }
      if (lo < len && __ldg(&cols[lo]) == c) {
        out[k] = b + lo;
      } else {
        out[k] = -1;
        atomicAdd(missing, 1);
      }
    }
  }
}

__global__ void scatter_add_kernel(long total, const double* __restrict__ A,
                                   const long* __restrict__ pos, double* __restrict__ vals) {
  for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long p = __ldg(&pos[t]);
    if (p >= 0) atomicAdd(&vals[p], __ldg(&A[t]));
  }
}

// loc[t][k] = pos[t][k] - row_ptr[dof[t]]: the entry's offset inside its CSR row
__global__ void csr_row_offsets_kernel(long total, int n, const int* __restrict__ dof,
                                       const long* __restrict__ row_ptr,
                                       const long* __restrict__ pos, uint16_t* __restrict__ loc,
                                       int* __restrict__ bad) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long)gridDim.x * blockDim.x) {
    const long t = i / n;
    const long r = __ldg(&dof[t]);
    const long p = __ldg(&pos[i]), b = __ldg(&row_ptr[r]), len = __ldg(&row_ptr[r + 1]) - b;
    const long d = p - b;
    if (p < 0 || d < 0 || d >= len || d > 0xFFFF) {
      loc[i] = 0;
      atomicAdd(bad, 1);
    } else {
      loc[i] = (uint16_t)d;
    }
  }
}

// Atomic-free numeric assembly: one warp per CSR row r sums the element-matrix rows
// incident to it (inc[inc_ptr[r] .. inc_ptr[r+1]), element-row ids e*n + j) into a
// shared-memory copy of the row, in a fixed order (bit-reproducible), then writes the
// row once (coalesced).  The n entries of one element row land on distinct columns,
// so a warp applies one element row per step without conflicts; KPL = entries per lane.
// Up to U element rows are loaded ahead of their application (memory-level parallelism).
template <int KPL>
__global__ void __launch_bounds__(256)
    csr_gather_rows_kernel(long nrows, int n, int wpb, int maxlen, const long* __restrict__ row_ptr,
                           const long* __restrict__ inc_ptr, const int* __restrict__ inc,
                           const uint16_t* __restrict__ loc, const double* __restrict__ A,
                           int acc, double* __restrict__ vals) {
  constexpr int U = 4;
  extern __shared__ double rowbuf[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= wpb) return;
  double* buf = rowbuf + (size_t)warp * maxlen;
  for (long r = (long)blockIdx.x * wpb + warp; r < nrows; r += (long)gridDim.x * wpb) {
    const long b = __ldg(&row_ptr[r]);
    const int len = (int)(__ldg(&row_ptr[r + 1]) - b);
    for (int p = lane; p < len; p += 32) buf[p] = 0.0;
    __syncwarp();
    const long i1 = __ldg(&inc_ptr[r + 1]);
    for (long i = __ldg(&inc_ptr[r]); i < i1; i += U) {
      double v[U][KPL];
      int o[U][KPL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long t = i + u < i1 ? (long)__ldg(&inc[i + u]) : -1;
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          const int k = lane + 32 * kk;
          const bool ok = t >= 0 && k < n;
          v[u][kk] = ok ? __ldcs(&A[t * n + k]) : 0.0;
          o[u][kk] = ok ? (int)__ldg(&loc[t * n + k]) : -1;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk)
          if (o[u][kk] >= 0) buf[o[u][kk]] += v[u][kk];
        __syncwarp();
      }
    }
    for (int p = lane; p < len; p += 32) vals[b + p] = acc ? vals[b + p] + buf[p] : buf[p];
    __syncwarp();
  }
}

int grid_for(long work, int block) {
  const long want = (work + block - 1) / block;
  const long cap = 8L * num_sms() * (2048 / block);
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_csr_row_offsets(long E, int n, const int* dof, const long* row_ptr,
                                   const long* pos, uint16_t* loc, int* bad, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  const long total = E * (long)n * n;
  csr_row_offsets_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, n, dof, row_ptr, pos, loc, bad);
  return cudaGetLastError();
}

cudaError_t launch_csr_gather_rows(long nrows, int n, int maxlen, const long* row_ptr,
                                   const long* inc_ptr, const int* inc, const uint16_t* loc,
                                   const double* A, int acc, double* vals, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  if (n > 64 || maxlen <= 0) return cudaErrorInvalidValue;
  // warps per 256-thread block: as many row buffers as fit in 200 KB of shared memory
  const size_t rowb = sizeof(double) * (size_t)maxlen;
  const int wpb = (int)std::min<size_t>(8, (200u << 10) / rowb);
  if (wpb < 1) return cudaErrorInvalidValue;
  const size_t smem = rowb * wpb;
  const long want = (nrows + wpb - 1) / wpb;
  const long cap = 64L * num_sms();
  const int grid = (int)std::min(want, cap);
  if (n <= 32) {
    auto k = csr_gather_rows_kernel<1>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 256, smem, s>>>(nrows, n, wpb, maxlen, row_ptr, inc_ptr, inc, loc, A, acc, vals);
  } else {
    auto k = csr_gather_rows_kernel<2>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 256, smem, s>>>(nrows, n, wpb, maxlen, row_ptr, inc_ptr, inc, loc, A, acc, vals);
  }
  return cudaGetLastError();
}

cudaError_t launch_gather(long E, int ncoef, const double* V, const int* cells, const double* coef,
                          const int* coef_idx, double* coords, double* coeffs, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  gather_kernel<<<grid_for(E * (12 + ncoef), 256), 256, 0, s>>>(E, ncoef, V, cells, coef, coef_idx,
                                                               coords, coeffs);
  return cudaGetLastError();
}

cudaError_t launch_csr_positions(long E, int n, const int* dof, const long* row_ptr,
                                 const int* col_idx, long* pos, int* missing, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  csr_positions_kernel<<<grid_for(E * n, 128), 128, 0, s>>>(E, n, dof, row_ptr, col_idx, pos,
                                                            missing);
  return cudaGetLastError();
}

cudaError_t launch_scatter_add(long total, const double* A, const long* pos, double* vals,
                               cudaStream_t s) {
  if (total <= 0) return cudaSuccess;
  scatter_add_kernel<<<grid_for(total, 256), 256, 0, s>>>(total, A, pos, vals);
  return cudaGetLastError();
}

}  // namespace femgpu
