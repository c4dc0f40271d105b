// helm_quad.cu -- weighted Helmholtz element matrices in the QUADRATURE schedule.
//
//   A_jk = |det J| sum_q W_q f(x_q) (grad phi_j . grad phi_k + phi_j phi_k)(x_q)
//
// This is femopt's sharing-elimination schedule for the form (the plan its cost
// model picks when pre-evaluation is rejected, proj/src/sharing.cpp:409-607 and
// driver.cpp:47-106 with T_H below the reference tensor's size): per quadrature
// point the j-side operands are hoisted -- s_q = W_q |det| f(x_q) and the
// physical gradients g_j = K^T D phi_j(x_q) -- and every (j,k) pair accumulates
// s_q (g_j . g_k + B_qj B_qk).  The TENSOR schedule of the same form
// (helmholtz.cu, A_e = sum_alpha g_alpha S_alpha on DMMA) needs 59 k flops per
// P3 cell against this schedule's ~270 k; femgpu's AUTO schedule choice
// (capi.cu, rank_schedules) ranks the two by their flop and byte counts against
// the device's FP64 and HBM peaks and a measured efficiency, like femopt's
// theta_pre / theta_se triage.  This kernel is the measured alternative that
// ranking is checked against (tests/test_schedule.py, profiles/).
//
// Organisation: one CTA of 32 cells per SM slot; lane = cell (every shared
// memory access of a warp is 32 consecutive doubles, conflict-free), warp w =
// upper (J <= K) tile of TJ x TJ pairs (NS = 20: 15 tiles of 4 x 4).  Points are
// processed in chunks of QC: all threads build the chunk's records (s_q, g_j,
// B_qj per cell, cell-fastest), then every tile warp accumulates them.  The
// element matrices are staged in the record buffer (mirror of the upper tiles)
// and written by one TMA bulk copy per cell.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

namespace hq {
constexpr int CELLS = 32;
constexpr int QC = 4;  // quadrature points per chunk
}  // namespace hq

template <int NS>
struct HelmQuadShape {
  static constexpr int TJ = NS % 4 == 0 ? 4 : 2;
  static constexpr int NB = NS / TJ;
  static constexpr int NTILE = NB * (NB + 1) / 2;
  static constexpr int WARPS = NTILE > 16 ? NTILE : 16;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int RECJ = 4 * hq::CELLS;                  // per (q, j): g0 g1 g2 B
  static constexpr int RECQ = NS * RECJ + hq::CELLS;          // + s_q
  static constexpr int REC_DBL = hq::QC * RECQ;
  static constexpr int CSTR = NS * NS + 2;                    // staging cell stride (16 B aligned;
                                                              // lane = cell: 4-way, not 32-way)
  static constexpr int STG_DBL = hq::CELLS * CSTR;            // staging (aliases the records)
  static constexpr int BODY = REC_DBL > STG_DBL ? REC_DBL : STG_DBL;
  static constexpr int CELLD = 10;                            // K(9), |det|
  static_assert(NS % TJ == 0, "tile size");
};

template <int NS>
size_t helm_quad_smem(int nc) {
  using Sh = HelmQuadShape<NS>;
  return sizeof(double) * ((size_t)Sh::BODY + hq::CELLS * (12 + nc) + hq::CELLS * Sh::CELLD);
}

// tab = [W(Q) | B(Q,NS) | D(3,Q,NS) | P(Q,NC)]
template <int NS>
__global__ void __launch_bounds__(HelmQuadShape<NS>::THREADS, 1)
    helm_quad_kernel(long E, int Q, int NC, const double* __restrict__ coords,
                     const double* __restrict__ coef, const double* __restrict__ tab,
                     double* __restrict__ A, int acc) {
  using Sh = HelmQuadShape<NS>;
  constexpr int CELLS = hq::CELLS, QC = hq::QC, TJ = Sh::TJ;
  extern __shared__ __align__(16) double smem[];
  double* sRec = smem;                       // [QC][NS][4][CELLS] | [QC][CELLS] s_q; staging after
  double* sIn = smem + Sh::BODY;             // [CELLS][12] | [CELLS][NC]
  double* sCell = sIn + CELLS * (12 + NC);   // [CELLS][CELLD]
  const double* gW = tab;
  const double* gB = gW + Q;
  const double* gD = gB + (size_t)Q * NS;
  const double* gP = gD + (size_t)3 * Q * NS;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // this warp's tile (J <= K), row-major over the upper triangle
  int TJi = 0, TKi = 0;
  {
    int t = warp;
    for (int J = 0; J < Sh::NB; ++J) {
      const int len = Sh::NB - J;
      if (t < len) {
        TJi = J;
        TKi = J + t;
        break;
      }
      t -= len;
    }
  }
  const bool tile_warp = warp < Sh::NTILE;
  const bool diag = TJi == TKi;
  const int j0 = TJi * TJ, k0 = TKi * TJ;
  const long ntiles = (E + CELLS - 1) / CELLS;

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = tile * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    __syncthreads();  // previous tile: staging read by its bulk stores, inputs consumed
    if (tid == 0) bulk_wait_read0();
    __syncthreads();
    for (int i = tid; i < nt * 12; i += Sh::THREADS) sIn[i] = coords[c0 * 12 + i];
    for (int i = tid; i < nt * NC; i += Sh::THREADS) sIn[CELLS * 12 + i] = coef[c0 * NC + i];
    __syncthreads();
    if (tid < CELLS) {
      double x[12];
#pragma unroll
      for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
        x[r] = tid < nt ? sIn[tid * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
      const Geo geo = cell_geometry(x);
      double* cd = sCell + tid * Sh::CELLD;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) cd[a * 3 + b] = geo.K[a][b];
      cd[9] = geo.adet;
    }
    double a[TJ][TJ];
#pragma unroll
    for (int x = 0; x < TJ; ++x)
#pragma unroll
      for (int y = 0; y < TJ; ++y) a[x][y] = 0.0;

    for (int q0 = 0; q0 < Q; q0 += QC) {
      const int qn = min(QC, Q - q0);
      __syncthreads();  // geometry visible / previous chunk's records consumed
      // ---- records of the chunk: one (cell, point, j-group) task per thread ----
      constexpr int JG = NS / 4 > 0 ? 4 : 1;        // j per task
      constexpr int NJG = (NS + JG - 1) / JG;
      for (int task = tid; task < CELLS * QC * NJG; task += Sh::THREADS) {
        const int c = task % CELLS, r = task / CELLS;
        const int ql = r % QC, jg = r / QC;
        if (ql >= qn) continue;
        const int q = q0 + ql;
        const double* cd = sCell + c * Sh::CELLD;
        double* rq = sRec + ql * Sh::RECQ;
        if (jg == 0) {
          double f = 0.0;  // f(x_q) = sum_m f_m P_m(x_q)
          const double* cf = sIn + CELLS * 12 + c * NC;
          for (int m = 0; m < NC; ++m) f += (c < nt ? cf[m] : 0.0) * __ldg(&gP[(size_t)q * NC + m]);
          rq[NS * Sh::RECJ + c] = __ldg(&gW[q]) * cd[9] * f;
        }
        double K[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) K[i] = cd[i];
#pragma unroll
        for (int jj = 0; jj < JG; ++jj) {
          const int j = jg * JG + jj;
          if (j >= NS) break;
          const double d0 = __ldg(&gD[((size_t)0 * Q + q) * NS + j]);
          const double d1 = __ldg(&gD[((size_t)1 * Q + q) * NS + j]);
          const double d2 = __ldg(&gD[((size_t)2 * Q + q) * NS + j]);
          double* rr = rq + j * Sh::RECJ + c;
#pragma unroll
          for (int b = 0; b < 3; ++b) rr[b * CELLS] = K[0 * 3 + b] * d0 + K[1 * 3 + b] * d1 + K[2 * 3 + b] * d2;
          rr[3 * CELLS] = __ldg(&gB[(size_t)q * NS + j]);
        }
      }
      __syncthreads();
      // ---- accumulate: warp = tile, lane = cell ----
      if (tile_warp) {
        for (int ql = 0; ql < qn; ++ql) {
          const double* rq = sRec + ql * Sh::RECQ + lane;
          const double s = rq[NS * Sh::RECJ];
          double gk[TJ][4];
#pragma unroll
          for (int y = 0; y < TJ; ++y)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) gk[y][cc] = rq[(k0 + y) * Sh::RECJ + cc * CELLS];
#pragma unroll
          for (int x = 0; x < TJ; ++x) {
            double gj[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) gj[cc] = s * rq[(j0 + x) * Sh::RECJ + cc * CELLS];
#pragma unroll
            for (int y = 0; y < TJ; ++y)
              a[x][y] = fma(gj[0], gk[y][0],
                            fma(gj[1], gk[y][1], fma(gj[2], gk[y][2], fma(gj[3], gk[y][3], a[x][y]))));
          }
        }
      }
    }
    __syncthreads();  // records consumed: the buffer becomes the staging area
    if (tile_warp) {
      double* stg = sRec + (size_t)lane * Sh::CSTR;
#pragma unroll
      for (int x = 0; x < TJ; ++x)
#pragma unroll
        for (int y = 0; y < TJ; ++y) {
          if (diag && y < x) continue;  // lower half of a diagonal tile: the mirror
          stg[(j0 + x) * NS + k0 + y] = a[x][y];
          stg[(k0 + y) * NS + j0 + x] = a[x][y];
        }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      for (int c = 0; c < nt; ++c) {
        double* dst = A + (c0 + c) * (size_t)NS * NS;
        if (acc)
          bulk_s2g_add(dst, sRec + (size_t)c * Sh::CSTR, NS * NS * 8);
        else
          bulk_s2g(dst, sRec + (size_t)c * Sh::CSTR, NS * NS * 8);
      }
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait0();
}

bool helm_quad_supported(int ns, int nc) { return (ns == 20 || ns == 10 || ns == 4) && nc > 0; }

size_t helm_quad_table_doubles(int nq, int ns, int nc) {
  return (size_t)nq * (1 + ns + 3 * ns + nc);
}

template <int NS>
static cudaError_t launch_hq(long E, int nq, int nc, const double* coords, const double* coef,
                             const double* tab, double* A, int acc, cudaStream_t s) {
  using Sh = HelmQuadShape<NS>;
  auto kern = helm_quad_kernel<NS>;
  const size_t smem = helm_quad_smem<NS>(nc);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  static const char once_key = 0;
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + hq::CELLS - 1) / hq::CELLS;
  const long nsm = num_sms();
  const int grid = (int)(ntiles < nsm ? ntiles : nsm);
  kern<<<grid, Sh::THREADS, smem, s>>>(E, nq, nc, coords, coef, tab, A, acc);
  return cudaGetLastError();
}

cudaError_t launch_helm_quad(int ns, int nq, int nc, long E, const double* coords,
                             const double* coef, const double* tab, double* A, int acc,
                             cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  if (ns == 20) return launch_hq<20>(E, nq, nc, coords, coef, tab, A, acc, s);
  if (ns == 10) return launch_hq<10>(E, nq, nc, coords, coef, tab, A, acc, s);
  if (ns == 4) return launch_hq<4>(E, nq, nc, coords, coef, tab, A, acc, s);
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
