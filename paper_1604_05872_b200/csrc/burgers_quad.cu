// burgers_quad.cu -- Burgers Jacobian (config 5) in the QUADRATURE schedule.
//
//   A_{(c,j),(d,k)} = sum_q s_q [ phi_j phi_k (d_d u_c + d_cd / dt)
//                                 + d_cd (phi_j (u.g_k) + nu g_j.g_k) ],   s_q = W_q |det J|
//
// femopt's sharing-elimination schedule for the form (proj/src/sharing.cpp:409-607):
// per cell and quadrature point the operands that depend on the point only --
// s_q, u(x_q), grad u(x_q) -- are hoisted, then every (j,k) pair accumulates its
// ten sums (the nine d_d u_c blocks and the scalar convection / diffusion / mass
// term).  It is the measured alternative to burgers.cu's TENSOR schedule (two DMMA
// GEMMs over pre-evaluated reference tensors); femgpu's cost model ranks the two
// (capi.cu, rank_schedules; profiles/schedule_choice_r02.json).
//
// Organisation: one warp per cell, lane k = basis function k of the trial side
// (lanes 20..31 idle: they compute clamped copies and store nothing); per cell the
// warp first tabulates the point data (s, u, grad u) of all Q points into shared
// memory (lane = point), then runs the j rows in groups of 4: lane k accumulates
// (j, k) for the group's four j over every point (40 accumulators), g_j and phi_j
// come from lane j by warp shuffles, and the group's rows (c, j) of A_e are written
// straight to HBM -- for each (c, j, d) the 20 lanes store 160 contiguous bytes.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {
namespace {

constexpr int BQ_NS = 20, BQ_N = 60;
constexpr int BQ_WARPS = 12;                // cells per CTA, one per warp (one CTA per SM)
constexpr int BQ_THREADS = 32 * BQ_WARPS;
constexpr int BQ_JG = 4;                    // j rows per pass
constexpr int BQ_PD = 13;                   // point data: s, u (3), grad u (9)

constexpr int BQ_CELLD = 12 + 3 * BQ_NS;    // coords | u dofs
// doubles of one warp's shared memory: point data of its cell, then its inputs
__host__ __device__ constexpr int bq_warp_dbl(int Q) { return (Q * BQ_PD + BQ_CELLD + 1) / 2 * 2; }

// tab = W(Q) | B(Q, NS) | D(3, Q, NS)
__global__ void __launch_bounds__(BQ_THREADS, 1)
    burgers_quad_kernel(long E, int Q, const double* __restrict__ coords,
                        const double* __restrict__ u, const double* __restrict__ tab, double nu,
                        double dt, double* __restrict__ A, int acc) {
  constexpr int NS = BQ_NS, N = BQ_N;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* pts = smem + warp * bq_warp_dbl(Q);  // [Q][PD]
  double* cd = pts + Q * BQ_PD;                // coords (12) | u (60)
  const double* gW = tab;
  const double* gB = gW + Q;
  const double* gD = gB + (size_t)Q * NS;
  const double rdt = 1.0 / dt;
  const int k = lane < NS ? lane : NS - 1;   // idle lanes mirror the last basis function

  for (long cell = (long)blockIdx.x * BQ_WARPS + warp; cell < E;
       cell += (long)gridDim.x * BQ_WARPS) {
    __syncwarp();  // previous cell's point data consumed
    for (int i = lane; i < 12; i += 32) cd[i] = coords[cell * 12 + i];
    for (int i = lane; i < 3 * NS; i += 32) cd[12 + i] = u[cell * 3 * NS + i];
    __syncwarp();
    double K[9], adet;
    {
      const Geo geo = cell_geometry(cd);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) K[a * 3 + b] = geo.K[a][b];
      adet = geo.adet;
    }
    // ---- point data, lane = point: s, u(x_q), grad u(x_q) ----
    for (int q = lane; q < Q; q += 32) {
      double uq[3] = {0, 0, 0}, gu[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      for (int m = 0; m < NS; ++m) {
        const double bm = __ldg(&gB[(size_t)q * NS + m]);
        const double d0 = __ldg(&gD[((size_t)0 * Q + q) * NS + m]);
        const double d1 = __ldg(&gD[((size_t)1 * Q + q) * NS + m]);
        const double d2 = __ldg(&gD[((size_t)2 * Q + q) * NS + m]);
        double g[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) g[b] = K[0 * 3 + b] * d0 + K[1 * 3 + b] * d1 + K[2 * 3 + b] * d2;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double um = cd[12 + c * NS + m];
          uq[c] = fma(um, bm, uq[c]);
#pragma unroll
          for (int d = 0; d < 3; ++d) gu[c][d] = fma(um, g[d], gu[c][d]);
        }
      }
      double* pq = pts + q * BQ_PD;
      pq[0] = __ldg(&gW[q]) * adet;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        pq[1 + c] = uq[c];
#pragma unroll
        for (int d = 0; d < 3; ++d) pq[4 + 3 * c + d] = gu[c][d];
      }
    }
    __syncwarp();
    // ---- rows in groups of BQ_JG: lane k accumulates (j, k) over the points ----
    double* Ac = A + cell * (size_t)N * N;
#pragma unroll 1
    for (int j0 = 0; j0 < NS; j0 += BQ_JG) {
      double M[BQ_JG][9], C[BQ_JG];
#pragma unroll
      for (int x = 0; x < BQ_JG; ++x) {
        C[x] = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) M[x][i] = 0.0;
      }
#pragma unroll 1
      for (int q = 0; q < Q; ++q) {
        const double* pq = pts + q * BQ_PD;
        const double s = pq[0];
        const double phik = __ldg(&gB[(size_t)q * NS + k]);
        const double d0 = __ldg(&gD[((size_t)0 * Q + q) * NS + k]);
        const double d1 = __ldg(&gD[((size_t)1 * Q + q) * NS + k]);
        const double d2 = __ldg(&gD[((size_t)2 * Q + q) * NS + k]);
        double gk[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) gk[b] = K[0 * 3 + b] * d0 + K[1 * 3 + b] * d1 + K[2 * 3 + b] * d2;
        const double ugk = pq[1] * gk[0] + pq[2] * gk[1] + pq[3] * gk[2];
        double gu[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) gu[i] = pq[4 + i];
#pragma unroll
        for (int x = 0; x < BQ_JG; ++x) {
          const int j = j0 + x;
          const double phij = __shfl_sync(0xffffffffu, phik, j);
          const double gj0 = __shfl_sync(0xffffffffu, gk[0], j);
          const double gj1 = __shfl_sync(0xffffffffu, gk[1], j);
          const double gj2 = __shfl_sync(0xffffffffu, gk[2], j);
          const double sj = s * phij;
          const double t = sj * phik;
#pragma unroll
          for (int i = 0; i < 9; ++i) M[x][i] = fma(t, gu[i], M[x][i]);
          const double dif = gj0 * gk[0] + gj1 * gk[1] + gj2 * gk[2];
          C[x] = fma(t, rdt, fma(sj, ugk, fma(s * nu, dif, C[x])));
        }
      }
      if (lane < NS) {
#pragma unroll
        for (int x = 0; x < BQ_JG; ++x)
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double v = M[x][3 * c + d] + (c == d ? C[x] : 0.0);
              double* p = Ac + (size_t)(c * NS + j0 + x) * N + d * NS + k;
              *p = acc ? *p + v : v;
            }
      }
    }
  }
}

size_t bq_smem(int nq) { return sizeof(double) * (size_t)BQ_WARPS * bq_warp_dbl(nq); }

}  // namespace

bool burgers_quad_supported(int nq, int ns) {
  return ns == BQ_NS && nq > 0 && bq_smem(nq) <= 227 * 1024;
}

cudaError_t launch_burgers_quad(int nq, int ns, long E, const double* coords, const double* coef,
                                const double* tab, double nu, double dt, double* A, int acc,
                                cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  if (!burgers_quad_supported(nq, ns)) return cudaErrorInvalidValue;
  static const char once_key = 0;
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    return cudaFuncSetAttribute(burgers_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                227 * 1024);
  });
  if (e0 != cudaSuccess) return e0;
  const long ctas = (E + BQ_WARPS - 1) / BQ_WARPS;
  const long maxc = num_sms();
  const int grid = (int)(ctas < maxc ? ctas : maxc);
  burgers_quad_kernel<<<grid, BQ_THREADS, bq_smem(nq), s>>>(E, nq, coords, coef, tab, nu, dt, A,
                                                           acc);
  return cudaGetLastError();
}

}  // namespace femgpu
