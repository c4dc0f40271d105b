// pair.cu -- vector-P_k element kernels on the FP64 CUDA cores (configs 3, 4).
//
// Linear elasticity   a(u,v) = int 2 mu eps(u):eps(v) + lam div u div v
// St Venant-Kirchhoff a(du,v) = int (grad du S + F dS[du]) : grad v
//
// Schedule: femopt's QUADRATURE choice for these forms (SURVEY.md §8a a5:
// "Elasticity per block at Q=8: none pre-evaluated; sharing elimination
// wins", App. A P13).  Sharing elimination (proj/src/sharing.cpp:409-607)
// hoists, per quadrature point, the operands that depend on one linear index
// only; we do the same, cut for the GPU:
//
//  * per quadrature point q and basis function j, a record of j-side operands
//    (elasticity: u_j = mu' g_j, v_j = lam' g_j, g_j;  SVK: s_j = w' S g_j,
//    lam' h_j, mu' h_j, mu' g_j, g_j, h_j = F g_j), computed once per (cell,j)
//    instead of once per (j,k) pair;
//  * every (c,d) component block of a (j,k) pair is a rank-2/3 update of these
//    records (component-blocked vector basis: the zero padding of the FFC
//    tables, zeroskip.cpp's concept, never enters the arithmetic);
//  * A_e is symmetric for both forms: only j<=k pairs are accumulated (2x2
//    register tiles over the upper triangle), mirrored in the epilogue;
//  * the records of point q+1 are computed in the same phase as the
//    accumulation of point q (double buffer), hiding their latency;
//  * element matrices are staged through shared memory 4 cells at a time and
//    written with coalesced 16-byte stores.
#include "common.cuh"
#include "femgpu_internal.h"
#include "../../include/femgpu.h"

namespace femgpu {

template <int KIND, int NS, int Q>
struct PairShape {
  static constexpr int N = 3 * NS;                       // element matrix N x N
  static constexpr int NJ = NS / 2;                      // 2-wide j/k groups
  static constexpr int NTILE = NJ * (NJ + 1) / 2;        // 2x2 tiles on/above the diagonal
  static constexpr int CELLS = 16;                       // cells per CTA tile
  static constexpr int THREADS = 256;
  static constexpr bool SVK = (KIND == FEMGPU_HYPERELASTICITY);
  static constexpr int NCOEF = SVK ? 3 * NS + 8 : 8;
  static constexpr int REC = SVK ? 18 : 10;              // j-record doubles
  // cell stride of a record buffer: (stride/2) odd -> conflict-free LDS.128
  static constexpr int RS0 = NS * REC + (SVK ? 6 : 0);
  static constexpr int RSTRIDE = ((RS0 / 2) % 2 == 1) ? RS0 : RS0 + 2;
  static constexpr int QD = 26;                          // SVK per-(cell,q) scalars
  static constexpr int TAB = Q + 3 * Q * NS + 4 * Q;     // W | D | P
  static constexpr int CELLD = 12 + 10 + NCOEF;          // coords | K(9), adet | coeffs
  static constexpr int OUT_CELLS = 4;                    // epilogue staging round
  static constexpr int RECBUF = 2 * CELLS * RSTRIDE;
  static constexpr int STG = OUT_CELLS * N * N;
  static constexpr int UNION = RECBUF > STG ? RECBUF : STG;
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)TAB + CELLS * CELLD + (SVK ? CELLS * Q * QD : 0) + UNION);
  static_assert(NS % 2 == 0, "2x2 tiling needs an even number of scalar dofs");
  static_assert(CELLS * NTILE <= THREADS, "one (cell, tile) per thread");
};

template <int KIND, int NS, int Q>
__global__ void __launch_bounds__(256, 1)
    pair_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                const double* __restrict__ tab, double* __restrict__ A, int acc) {
  using Sh = PairShape<KIND, NS, Q>;
  constexpr int N = Sh::N;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;
  double* sD = sW + Q;            // [3][Q][NS]
  double* sP = sD + 3 * Q * NS;   // [Q][4]
  double* sCell = smem + Sh::TAB; // [CELLS][CELLD]
  double* sQ = sCell + Sh::CELLS * Sh::CELLD;                 // SVK: [CELLS][Q][QD]
  double* sU = sQ + (Sh::SVK ? Sh::CELLS * Q * Sh::QD : 0);   // records / staging

  const int tid = threadIdx.x;
  for (int i = tid; i < Sh::TAB; i += Sh::THREADS) smem[i] = tab[i];

  // (cell, tile) owned in the accumulation phase
  const int my_cell = tid % Sh::CELLS;
  const int my_tile = tid / Sh::CELLS;
  const bool active = my_tile < Sh::NTILE;
  int TJ = 0, TK = 0;
  {
    int t = active ? my_tile : 0;
    for (int J = 0; J < Sh::NJ; ++J) {
      int len = Sh::NJ - J;
      if (t < len) { TJ = J; TK = J + t; break; }
      t -= len;
    }
  }
  const int j0 = 2 * TJ, k0 = 2 * TK;

  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = tile * Sh::CELLS;
    const int nt = (int)min((long)Sh::CELLS, E - c0);
    __syncthreads();  // previous epilogue done with sCell / staging
    // ---- load raw inputs (coalesced) ---------------------------------------
    for (int i = tid; i < Sh::CELLS * 12; i += Sh::THREADS) {
      const int c = i / 12, r = i % 12;
      // cells past the end get the reference tet (finite geometry, never stored)
      const double ref = (r == 3 || r == 7 || r == 11) ? 1.0 : 0.0;
      sCell[c * Sh::CELLD + r] = c < nt ? coords[(c0 + c) * 12 + r] : ref;
    }
    for (int i = tid; i < Sh::CELLS * Sh::NCOEF; i += Sh::THREADS) {
      const int c = i / Sh::NCOEF, r = i % Sh::NCOEF;
      sCell[c * Sh::CELLD + 22 + r] = c < nt ? coef[(c0 + c) * Sh::NCOEF + r] : 0.0;
    }
    __syncthreads();
    if (tid < Sh::CELLS) {
      double* cd = sCell + tid * Sh::CELLD;
      const Geo g = cell_geometry(cd);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) cd[12 + a * 3 + b] = g.K[a][b];
      cd[21] = g.adet;
    }
    __syncthreads();
    if constexpr (Sh::SVK) {
      // ---- per (cell, q): F, w' S, F F^T, lam', mu' (St Venant-Kirchhoff) --
      for (int task = tid; task < Sh::CELLS * Q; task += Sh::THREADS) {
        const int c = task / Q, q = task % Q;
        const double* cd = sCell + c * Sh::CELLD;
        const double* K = cd + 12;
        const double* w = cd + 22;              // [3][NS]
        const double* mu = cd + 22 + 3 * NS;
        const double* lam = mu + 4;
        double muq = 0, lamq = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          muq += mu[m] * sP[q * 4 + m];
          lamq += lam[m] * sP[q * 4 + m];
        }
        const double wq = sW[q] * cd[21];
        double F[3][3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          double gr[3] = {0, 0, 0};  // reference gradient of w_cc
#pragma unroll
          for (int m = 0; m < NS; ++m) {
            const double wm = w[cc * NS + m];
#pragma unroll
            for (int a = 0; a < 3; ++a) gr[a] += wm * sD[(a * Q + q) * NS + m];
          }
#pragma unroll
          for (int b = 0; b < 3; ++b)
            F[cc][b] = (cc == b ? 1.0 : 0.0) + gr[0] * K[0 * 3 + b] + gr[1] * K[1 * 3 + b] +
                       gr[2] * K[2 * 3 + b];
        }
        double Ee[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double t = F[0][a] * F[0][b] + F[1][a] * F[1][b] + F[2][a] * F[2][b];
            Ee[a][b] = 0.5 * (a == b ? t - 1.0 : t);
          }
        const double trE = Ee[0][0] + Ee[1][1] + Ee[2][2];
        double* qd = sQ + (c * Q + q) * Sh::QD;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            qd[a * 3 + b] = F[a][b];
            qd[9 + a * 3 + b] = wq * ((a == b ? lamq * trE : 0.0) + 2.0 * muq * Ee[a][b]);
          }
        const int ab[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          const int a = ab[s][0], b = ab[s][1];
          qd[18 + s] = F[a][0] * F[b][0] + F[a][1] * F[b][1] + F[a][2] * F[b][2];
        }
        qd[24] = lamq * wq;
        qd[25] = muq * wq;
      }
      __syncthreads();
    }

    // ---- per-(cell, j) records of point q -> buffer q&1 ---------------------
    auto make_records = [&](int q) {
      if (tid >= Sh::CELLS * NS) return;
      const int c = tid / NS, j = tid % NS;
      const double* cd = sCell + c * Sh::CELLD;
      const double* K = cd + 12;
      double* rec = sU + (q & 1) * Sh::CELLS * Sh::RSTRIDE + c * Sh::RSTRIDE + j * Sh::REC;
      double g[3];
#pragma unroll
      for (int b = 0; b < 3; ++b)
        g[b] = K[0 * 3 + b] * sD[(0 * Q + q) * NS + j] + K[1 * 3 + b] * sD[(1 * Q + q) * NS + j] +
               K[2 * 3 + b] * sD[(2 * Q + q) * NS + j];
      if constexpr (!Sh::SVK) {
        const double* mu = cd + 22;
        const double* lam = cd + 26;
        double muq = 0, lamq = 0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          muq += mu[m] * sP[q * 4 + m];
          lamq += lam[m] * sP[q * 4 + m];
        }
        const double wq = sW[q] * cd[21];
        const double mq = muq * wq, lq = lamq * wq;
        double2* r2 = reinterpret_cast<double2*>(rec);
        r2[0] = make_double2(mq * g[0], mq * g[1]);
        r2[1] = make_double2(mq * g[2], lq * g[0]);
        r2[2] = make_double2(lq * g[1], lq * g[2]);
        r2[3] = make_double2(g[0], g[1]);
        rec[8] = g[2];
      } else {
        const double* qd = sQ + (c * Q + q) * Sh::QD;
        double h[3], s[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          h[a] = qd[a * 3 + 0] * g[0] + qd[a * 3 + 1] * g[1] + qd[a * 3 + 2] * g[2];
          s[a] = qd[9 + a * 3 + 0] * g[0] + qd[9 + a * 3 + 1] * g[1] + qd[9 + a * 3 + 2] * g[2];
        }
        const double lq = qd[24], mq = qd[25];
        double2* r2 = reinterpret_cast<double2*>(rec);
        r2[0] = make_double2(s[0], s[1]);
        r2[1] = make_double2(s[2], lq * h[0]);
        r2[2] = make_double2(lq * h[1], lq * h[2]);
        r2[3] = make_double2(mq * h[0], mq * h[1]);
        r2[4] = make_double2(mq * h[2], mq * g[0]);
        r2[5] = make_double2(mq * g[1], mq * g[2]);
        r2[6] = make_double2(g[0], g[1]);
        r2[7] = make_double2(g[2], h[0]);
        r2[8] = make_double2(h[1], h[2]);
        if (j == 0) {
          double* ff = sU + (q & 1) * Sh::CELLS * Sh::RSTRIDE + c * Sh::RSTRIDE + NS * Sh::REC;
#pragma unroll
          for (int i = 0; i < 6; ++i) ff[i] = qd[18 + i];
        }
      }
    };

    double a4[2][2][3][3];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) a4[x][y][c][d] = 0.0;

    make_records(0);
    __syncthreads();
#pragma unroll 1
    for (int q = 0; q < Q; ++q) {
      if (q + 1 < Q) make_records(q + 1);
      if (active) {
        const double* base = sU + (q & 1) * Sh::CELLS * Sh::RSTRIDE + my_cell * Sh::RSTRIDE;
        if constexpr (!Sh::SVK) {
          double gk[2][3];
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            const double* r = base + (k0 + y) * Sh::REC;
            const double2 p0 = *reinterpret_cast<const double2*>(r + 6);
            gk[y][0] = p0.x; gk[y][1] = p0.y; gk[y][2] = r[8];
          }
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const double* r = base + (j0 + x) * Sh::REC;
            const double2 p0 = *reinterpret_cast<const double2*>(r);
            const double2 p1 = *reinterpret_cast<const double2*>(r + 2);
            const double2 p2 = *reinterpret_cast<const double2*>(r + 4);
            const double u[3] = {p0.x, p0.y, p1.x}, v[3] = {p1.y, p2.x, p2.y};
#pragma unroll
            for (int y = 0; y < 2; ++y) {
              const double S = u[0] * gk[y][0] + u[1] * gk[y][1] + u[2] * gk[y][2];
#pragma unroll
              for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int d = 0; d < 3; ++d)
                  a4[x][y][c][d] = fma(u[d], gk[y][c], fma(v[c], gk[y][d], a4[x][y][c][d]));
#pragma unroll
              for (int c = 0; c < 3; ++c) a4[x][y][c][c] += S;
            }
          }
        } else {
          double gk[2][3], hk[2][3];
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            const double* r = base + (k0 + y) * Sh::REC;
            const double2 p0 = *reinterpret_cast<const double2*>(r + 12);
            const double2 p1 = *reinterpret_cast<const double2*>(r + 14);
            const double2 p2 = *reinterpret_cast<const double2*>(r + 16);
            gk[y][0] = p0.x; gk[y][1] = p0.y; gk[y][2] = p1.x;
            hk[y][0] = p1.y; hk[y][1] = p2.x; hk[y][2] = p2.y;
          }
          const double* ffp = base + NS * Sh::REC;
          const double ff[3][3] = {{ffp[0], ffp[1], ffp[2]}, {ffp[1], ffp[3], ffp[4]},
                                   {ffp[2], ffp[4], ffp[5]}};
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const double* r = base + (j0 + x) * Sh::REC;
            double rv[12];
#pragma unroll
            for (int i = 0; i < 6; ++i) {
              const double2 p = *reinterpret_cast<const double2*>(r + 2 * i);
              rv[2 * i] = p.x;
              rv[2 * i + 1] = p.y;
            }
            const double* s = rv;       // w' S g_j
            const double* lh = rv + 3;  // lam' h_j
            const double* mh = rv + 6;  // mu' h_j
            const double* mg = rv + 9;  // mu' g_j
#pragma unroll
            for (int y = 0; y < 2; ++y) {
              const double t1 = s[0] * gk[y][0] + s[1] * gk[y][1] + s[2] * gk[y][2];
              const double t2 = mg[0] * gk[y][0] + mg[1] * gk[y][1] + mg[2] * gk[y][2];
#pragma unroll
              for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int d = 0; d < 3; ++d)
                  a4[x][y][c][d] =
                      fma(lh[c], hk[y][d], fma(hk[y][c], mh[d], fma(t2, ff[c][d], a4[x][y][c][d])));
#pragma unroll
              for (int c = 0; c < 3; ++c) a4[x][y][c][c] += t1;
            }
          }
        }
      }
      __syncthreads();
    }

    // ---- epilogue: mirror into staging, 4 cells per round, coalesced stores --
    double* stg = sU;
#pragma unroll 1
    for (int r = 0; r < Sh::CELLS / Sh::OUT_CELLS; ++r) {
      const int lc = my_cell - r * Sh::OUT_CELLS;
      if (active && lc >= 0 && lc < Sh::OUT_CELLS) {
        double* As = stg + lc * N * N;
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y) {
            const int j = j0 + x, k = k0 + y;
            if (j > k) continue;
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                const double v = a4[x][y][c][d];
                As[(c * NS + j) * N + d * NS + k] = v;
                As[(d * NS + k) * N + c * NS + j] = v;
              }
          }
      }
      __syncthreads();
      const long cb = c0 + r * Sh::OUT_CELLS;
      const int ncell = (int)max(0L, min((long)Sh::OUT_CELLS, E - cb));
      double2* gA = reinterpret_cast<double2*>(A + cb * N * N);
      const double2* s2 = reinterpret_cast<const double2*>(stg);
      for (int i = tid; i < ncell * N * N / 2; i += Sh::THREADS) {
        double2 v = s2[i];
        if (acc) {
          double2 o = gA[i];
          v.x += o.x;
          v.y += o.y;
        }
        stg_stream(gA + i, v);
      }
      __syncthreads();
    }
  }
}

template <int KIND, int NS, int Q>
static cudaError_t launch_pair_t(long E, const double* coords, const double* coef,
                                 const double* tab, double* A, int acc, cudaStream_t s) {
  using Sh = PairShape<KIND, NS, Q>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(pair_kernel<KIND, NS, Q>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  const int grid = (int)(ntiles < (long)kNumSMs * 8 ? ntiles : (long)kNumSMs * 8);
  pair_kernel<KIND, NS, Q><<<grid, Sh::THREADS, Sh::SMEM, s>>>(E, coords, coef, tab, A, acc);
  return cudaGetLastError();
}

bool pair_supported(int kind, int nq, int ns) {
  if (ns != 10) return false;
  if (kind == FEMGPU_ELASTICITY) return nq == 8 || nq == 27;
  if (kind == FEMGPU_HYPERELASTICITY) return nq == 27 || nq == 8;
  return false;
}

cudaError_t launch_pair(int kind, int nq, int ns, long E, const double* coords, const double* coef,
                        const double* tab, double* A, int acc, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  if (ns == 10) {
    if (kind == FEMGPU_ELASTICITY && nq == 8)
      return launch_pair_t<FEMGPU_ELASTICITY, 10, 8>(E, coords, coef, tab, A, acc, s);
    if (kind == FEMGPU_ELASTICITY && nq == 27)
      return launch_pair_t<FEMGPU_ELASTICITY, 10, 27>(E, coords, coef, tab, A, acc, s);
    if (kind == FEMGPU_HYPERELASTICITY && nq == 27)
      return launch_pair_t<FEMGPU_HYPERELASTICITY, 10, 27>(E, coords, coef, tab, A, acc, s);
    if (kind == FEMGPU_HYPERELASTICITY && nq == 8)
      return launch_pair_t<FEMGPU_HYPERELASTICITY, 10, 8>(E, coords, coef, tab, A, acc, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
