// pair.cu -- vector-P_k element kernels on the FP64 CUDA cores (configs 3, 4).
//
// Linear elasticity   a(u,v) = int 2 mu eps(u):eps(v) + lam div u div v
// St Venant-Kirchhoff a(du,v) = int (grad du S + F dS[du]) : grad v
//
// Schedule: femopt's QUADRATURE choice for these forms (SURVEY.md §8a a5:
// "Elasticity per block at Q=8: none pre-evaluated; sharing elimination
// wins", App. A P13).  Sharing elimination (proj/src/sharing.cpp:409-607)
// hoists, per quadrature point, the operands that depend on one linear index
// only; the same structure, cut for the GPU:
//
//  * per (cell, quadrature point q, basis function j) a record of j-side
//    operands -- g_j = K^T grad phi_j (elasticity), plus h_j = F g_j and
//    s_j = w' S g_j (St Venant-Kirchhoff) -- computed once for a chunk of
//    quadrature points, stored cell-fastest so the 8 lanes of one (j,k) tile
//    read consecutive addresses;
//  * every (c,d) component block of a (j,k) pair is a rank-2/3 update of these
//    records (component-blocked vector basis: the zero padding of the FFC
//    tables, zeroskip.cpp's concept, never enters the arithmetic):
//      elasticity  A(c,d) += mu' g_j[d] g_k[c] + lam' g_j[c] g_k[d] + d_cd mu' g_j.g_k
//      SVK         A(c,d) += lam' h_j[c] h_k[d] + mu' h_k[c] h_j[d]
//                            + mu' (F F^T)_cd g_j.g_k + d_cd s_j.g_k
//  * A_e is symmetric for both forms: only j<=k pairs are accumulated (2x2
//    register tiles over the upper triangle of the 10x10 (j,k) grid), one
//    (cell, tile) per thread, no synchronisation inside the q loop;
//  * the 8 element matrices of a tile (58 KB) are staged in shared memory
//    (cell stride 902 doubles: conflict-free 16-byte stores) and written to HBM
//    by TMA bulk copies (cp.async.bulk / cp.reduce.async.bulk .add.f64 for the
//    += contract), so no thread spends time on the store stream; the next
//    tile's inputs are prefetched
//    with cp.async while the current tile accumulates; 2-3 CTAs per SM overlap
//    one tile's store burst with another's arithmetic.
#include "common.cuh"
#include "femgpu_internal.h"
#include "../../include/femgpu.h"

namespace femgpu {

template <int KIND, int NS, int Q>
struct PairShape {
  static constexpr int N = 3 * NS;                       // element matrix N x N
  static constexpr int NJ = NS / 2;                      // 2-wide j/k groups
  static constexpr int NTILE = NJ * (NJ + 1) / 2;        // 2x2 tiles on/above the diagonal
  static constexpr int CELLS = 8;                        // cells per CTA tile
  static constexpr int THREADS = 128;                    // 8 cells x 16 tile slots
  static constexpr bool SVK = (KIND == FEMGPU_HYPERELASTICITY);
  static constexpr int CTAS_PER_SM = SVK ? 2 : 3;        // independent tiles overlap phases
  static constexpr int NCOEF = SVK ? 3 * NS + 8 : 8;
  static constexpr int QC = SVK ? 9 : Q;                 // quadrature points per chunk
  static constexpr int NCHUNK = (Q + QC - 1) / QC;
  static constexpr int RECD = SVK ? 9 : 3;               // per (q,j): g | h | s
  static constexpr int QSD = SVK ? 8 : 2;                // per q: lam', mu' | F F^T (6)
  static constexpr int QDD = 18;                         // SVK per (cell,q): F, w'S
  static constexpr int REC_DBL = QC * (NS * RECD + QSD) * CELLS;
  static constexpr int CSTRIDE = N * N + 2;              // staging stride: (stride/2) odd
  static constexpr int STG_DBL = CELLS * CSTRIDE;
  static constexpr int UNION = REC_DBL > STG_DBL ? REC_DBL : STG_DBL;
  static constexpr int TAB0 = Q + 3 * Q * NS + 4 * Q;    // W | D | P
  static constexpr int TAB = (TAB0 + 1) / 2 * 2;
  static constexpr int CELLD = 12 + 10;                  // coords | K(9), adet
  static constexpr int IN_DBL = CELLS * (12 + NCOEF);    // raw inputs (cp.async target)
  static constexpr int QD_DBL = SVK ? QC * CELLS * QDD : 0;
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)TAB + CELLS * CELLD + IN_DBL + QD_DBL + UNION);
  static_assert(NS % 2 == 0, "2x2 tiling needs an even number of scalar dofs");
  static_assert(CELLS * (NTILE + 1) <= THREADS, "one (cell, tile) per thread");
  static_assert((CSTRIDE / 2) % 2 == 1, "conflict-free staging stride");
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <int KIND, int NS, int Q>
__global__ void __launch_bounds__(128, PairShape<KIND, NS, Q>::CTAS_PER_SM)
    pair_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                const double* __restrict__ tab, double* __restrict__ A, int acc) {
  using Sh = PairShape<KIND, NS, Q>;
  constexpr int N = Sh::N, CELLS = Sh::CELLS;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;
  double* sD = sW + Q;                      // [3][Q][NS]
  double* sP = sD + 3 * Q * NS;             // [Q][4]
  double* sCell = smem + Sh::TAB;           // [CELLS][CELLD]
  double* sIn = sCell + CELLS * Sh::CELLD;  // [CELLS][12] | [CELLS][NCOEF]
  double* sQd = sIn + Sh::IN_DBL;           // SVK: [QC][CELLS][QDD]
  double* sU = sQd + Sh::QD_DBL;            // records (chunk) / output staging
  // record layout: rec[((ql*NS + j)*RECD + comp)*CELLS + cell], then per-q scalars
  double* sQs = sU + Sh::QC * NS * Sh::RECD * CELLS;  // [QC][QSD][CELLS]

  const int tid = threadIdx.x;
  for (int i = tid; i < Sh::TAB0; i += Sh::THREADS) smem[i] = tab[i];

  const int cell = tid % CELLS;
  const int my_tile = tid / CELLS;
  const bool active = my_tile < Sh::NTILE;
  int TJ = 0, TK = 0;
  {
    int t = active ? my_tile : 0;
    for (int J = 0; J < Sh::NJ; ++J) {
      const int len = Sh::NJ - J;
      if (t < len) {
        TJ = J;
        TK = J + t;
        break;
      }
      t -= len;
    }
  }
  const int j0 = 2 * TJ, k0 = 2 * TK;

  const long ntiles = (E + CELLS - 1) / CELLS;
  auto prefetch = [&](long tile) {
    const long c0 = tile * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    for (int i = tid; i < nt * 12; i += Sh::THREADS) cp_async8(&sIn[i], coords + c0 * 12 + i);
    for (int i = tid; i < nt * Sh::NCOEF; i += Sh::THREADS)
      cp_async8(&sIn[CELLS * 12 + i], coef + c0 * Sh::NCOEF + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if ((long)blockIdx.x < ntiles) prefetch(blockIdx.x);

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = tile * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (tid == 0) bulk_wait_read0();  // previous tile's bulk stores have read the staging
    __syncthreads();
    if (tid < CELLS) {
      double x[12];
#pragma unroll
      for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
        x[r] = tid < nt ? sIn[tid * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
      const Geo g = cell_geometry(x);
      double* cd = sCell + tid * Sh::CELLD;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) cd[12 + a * 3 + b] = g.K[a][b];
      cd[21] = g.adet;
    }
    __syncthreads();
    auto coefv = [&](int c, int r) -> double {
      return c < nt ? sIn[CELLS * 12 + c * Sh::NCOEF + r] : 0.0;
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

#pragma unroll 1
    for (int ch = 0; ch < Sh::NCHUNK; ++ch) {
      const int q0 = ch * Sh::QC;
      const int qn = min(Sh::QC, Q - q0);
      if constexpr (Sh::SVK) {
        // ---- per (cell, q): F = I + grad w, w' S, F F^T, lam', mu' ---------
        for (int task = tid; task < CELLS * qn; task += Sh::THREADS) {
          const int c = task % CELLS, ql = task / CELLS, q = q0 + ql;
          const double* cd = sCell + c * Sh::CELLD;
          const double* K = cd + 12;
          double muq = 0, lamq = 0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            muq += coefv(c, 3 * NS + m) * sP[q * 4 + m];
            lamq += coefv(c, 3 * NS + 4 + m) * sP[q * 4 + m];
          }
          const double wq = sW[q] * cd[21];
          double F[3][3];
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            double gr[3] = {0, 0, 0};  // reference gradient of w_cc
#pragma unroll
            for (int m = 0; m < NS; ++m) {
              const double wm = coefv(c, cc * NS + m);
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
          double* qd = sQd + (ql * CELLS + c) * Sh::QDD;
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              qd[a * 3 + b] = F[a][b];
              qd[9 + a * 3 + b] = wq * ((a == b ? lamq * trE : 0.0) + 2.0 * muq * Ee[a][b]);
            }
          double* qs = sQs + ql * Sh::QSD * CELLS + c;
          qs[0 * CELLS] = lamq * wq;
          qs[1 * CELLS] = muq * wq;
          // F F^T: (0,0),(0,1),(0,2),(1,1),(1,2),(2,2)
          qs[2 * CELLS] = F[0][0] * F[0][0] + F[0][1] * F[0][1] + F[0][2] * F[0][2];
          qs[3 * CELLS] = F[0][0] * F[1][0] + F[0][1] * F[1][1] + F[0][2] * F[1][2];
          qs[4 * CELLS] = F[0][0] * F[2][0] + F[0][1] * F[2][1] + F[0][2] * F[2][2];
          qs[5 * CELLS] = F[1][0] * F[1][0] + F[1][1] * F[1][1] + F[1][2] * F[1][2];
          qs[6 * CELLS] = F[1][0] * F[2][0] + F[1][1] * F[2][1] + F[1][2] * F[2][2];
          qs[7 * CELLS] = F[2][0] * F[2][0] + F[2][1] * F[2][1] + F[2][2] * F[2][2];
        }
        __syncthreads();
      }
      // ---- records of the chunk: per (cell, q, j) -------------------------
      for (int task = tid; task < CELLS * qn * NS; task += Sh::THREADS) {
        const int c = task % CELLS, r = task / CELLS;
        const int j = r % NS, ql = r / NS, q = q0 + ql;
        const double* cd = sCell + c * Sh::CELLD;
        const double* K = cd + 12;
        double g[3];
#pragma unroll
        for (int b = 0; b < 3; ++b)
          g[b] = K[0 * 3 + b] * sD[(0 * Q + q) * NS + j] + K[1 * 3 + b] * sD[(1 * Q + q) * NS + j] +
                 K[2 * 3 + b] * sD[(2 * Q + q) * NS + j];
        double* rec = sU + ((ql * NS + j) * Sh::RECD) * CELLS + c;
#pragma unroll
        for (int b = 0; b < 3; ++b) rec[b * CELLS] = g[b];
        if constexpr (Sh::SVK) {
          const double* qd = sQd + (ql * CELLS + c) * Sh::QDD;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            rec[(3 + a) * CELLS] = qd[a * 3 + 0] * g[0] + qd[a * 3 + 1] * g[1] + qd[a * 3 + 2] * g[2];
            rec[(6 + a) * CELLS] =
                qd[9 + a * 3 + 0] * g[0] + qd[9 + a * 3 + 1] * g[1] + qd[9 + a * 3 + 2] * g[2];
          }
        } else if (j == 0) {
          double muq = 0, lamq = 0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            muq += coefv(c, m) * sP[q * 4 + m];
            lamq += coefv(c, 4 + m) * sP[q * 4 + m];
          }
          const double wq = sW[q] * cd[21];
          double* qs = sQs + ql * Sh::QSD * CELLS + c;
          qs[0] = lamq * wq;
          qs[CELLS] = muq * wq;
        }
      }
      __syncthreads();
      if (ch == Sh::NCHUNK - 1 && tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);
      // ---- accumulate (no synchronisation inside) --------------------------
      if (active) {
#pragma unroll 1
        for (int ql = 0; ql < qn; ++ql) {
          const double* rq = sU + ql * NS * Sh::RECD * CELLS + cell;
          const double* qs = sQs + ql * Sh::QSD * CELLS + cell;
          const double lq = qs[0], mq = qs[CELLS];
          double gk[2][3];
#pragma unroll
          for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int b = 0; b < 3; ++b) gk[y][b] = rq[((k0 + y) * Sh::RECD + b) * CELLS];
          if constexpr (!Sh::SVK) {
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              double u[3], v[3];
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                const double gj = rq[((j0 + x) * Sh::RECD + b) * CELLS];
                u[b] = mq * gj;
                v[b] = lq * gj;
              }
              // independent FMA passes (no dependent pairs back to back)
#pragma unroll
              for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                  for (int d = 0; d < 3; ++d) a4[x][y][c][d] = fma(v[c], gk[y][d], a4[x][y][c][d]);
#pragma unroll
              for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                  for (int d = 0; d < 3; ++d) a4[x][y][c][d] = fma(u[d], gk[y][c], a4[x][y][c][d]);
#pragma unroll
              for (int y = 0; y < 2; ++y) {
                const double S = u[0] * gk[y][0] + u[1] * gk[y][1] + u[2] * gk[y][2];
#pragma unroll
                for (int c = 0; c < 3; ++c) a4[x][y][c][c] += S;
              }
            }
          } else {
            double hk[2][3];
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
              for (int b = 0; b < 3; ++b) hk[y][b] = rq[((k0 + y) * Sh::RECD + 3 + b) * CELLS];
            const double f00 = qs[2 * CELLS], f01 = qs[3 * CELLS], f02 = qs[4 * CELLS];
            const double f11 = qs[5 * CELLS], f12 = qs[6 * CELLS], f22 = qs[7 * CELLS];
            const double ff[3][3] = {{f00, f01, f02}, {f01, f11, f12}, {f02, f12, f22}};
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              double gj[3], lh[3], mh[3], s[3];
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                const double* r = rq + ((j0 + x) * Sh::RECD) * CELLS;
                gj[b] = mq * r[b * CELLS];           // mu' g_j
                const double h = r[(3 + b) * CELLS];
                lh[b] = lq * h;                      // lam' h_j
                mh[b] = mq * h;                      // mu' h_j
                s[b] = r[(6 + b) * CELLS];           // w' S g_j
              }
              double t1[2], t2[2];
#pragma unroll
              for (int y = 0; y < 2; ++y) {
                t1[y] = s[0] * gk[y][0] + s[1] * gk[y][1] + s[2] * gk[y][2];
                t2[y] = gj[0] * gk[y][0] + gj[1] * gk[y][1] + gj[2] * gk[y][2];
              }
              // independent FMA passes over the 18 accumulators of this j
#pragma unroll
              for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                  for (int d = 0; d < 3; ++d) a4[x][y][c][d] = fma(lh[c], hk[y][d], a4[x][y][c][d]);
#pragma unroll
              for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                  for (int d = 0; d < 3; ++d) a4[x][y][c][d] = fma(hk[y][c], mh[d], a4[x][y][c][d]);
#pragma unroll
              for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                  for (int d = 0; d < 3; ++d) a4[x][y][c][d] = fma(t2[y], ff[c][d], a4[x][y][c][d]);
#pragma unroll
              for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int c = 0; c < 3; ++c) a4[x][y][c][c] += t1[y];
            }
          }
        }
      }
      __syncthreads();  // records consumed (next chunk / staging overwrite them)
    }

    // ---- epilogue: mirror into staging (all 16 cells), coalesced stores -----
    double* stg = sU + cell * Sh::CSTRIDE;
    if (active) {
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const int j = j0 + x;
            // row (c, j), columns (d, k0..k0+1): one 16-byte store
            *reinterpret_cast<double2*>(&stg[(c * NS + j) * N + d * NS + k0]) =
                make_double2(a4[x][0][c][d], a4[x][1][c][d]);
          }
      if (TJ != TK) {
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const int k = k0 + y;
              // mirror: row (d, k), columns (c, j0..j0+1)
              *reinterpret_cast<double2*>(&stg[(d * NS + k) * N + c * NS + j0]) =
                  make_double2(a4[0][y][c][d], a4[1][y][c][d]);
            }
      } else {
        // diagonal tile: entry (j0+1, k0) is the mirror of (j0, k0+1)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d)
            stg[(d * NS + k0 + 1) * N + c * NS + j0] = a4[0][1][c][d];
      }
    }
    // staged element matrices -> global by the TMA engine (async bulk copies,
    // or bulk reductions for the += contract); threads move on immediately
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      for (int c = 0; c < nt; ++c) {
        double* dst = A + (c0 + c) * (size_t)N * N;
        if (acc)
          bulk_s2g_add(dst, sU + c * Sh::CSTRIDE, N * N * 8);
        else
          bulk_s2g(dst, sU + c * Sh::CSTRIDE, N * N * 8);
      }
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait0();
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
  const long maxc = (long)Sh::CTAS_PER_SM * kNumSMs;
  const int grid = (int)(ntiles < maxc ? ntiles : maxc);
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
