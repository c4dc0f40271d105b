// vector.cu -- element VECTORS (arity-1 forms) on the FP64 CUDA cores.
//
// The reference's validator admits arity-1 linear nests beside the bilinear ones
// (proj/src/kernel.cpp:369-390; the `linear_json` corpus kernel, kernels.hpp:250-259);
// paper_1604_05872_b200/ir.py writes them for the BASELINE families and the generic
// IR backend runs them.  These are the hand-written fast paths (femgpu_assemble_vector):
//
//   Helmholtz load      b_j     = int f phi_j
//                               = |det| sum_m M_jm f_m,  M_jm = sum_q W_q B_qj P_qm
//                                 (pre-evaluated on the host, preeval.cpp:269-274 order)
//   St Venant-Kirchhoff r_(c,j) = int (F S) : grad(phi_j e_c)
//                               = sum_q W_q |det| sum_a T_ca(q) D_a,qj,  T = (F S) K^T
//   Burgers             r_(c,j) = int (u_c/dt + (u.grad) u_c) phi_j + nu grad u_c . grad phi_j
//                               = sum_q W_q |det| (adv_c B_qj + sum_a t_ca D_a,qj),
//                                 t_ca = nu sum_b K_ab (grad u_c)_b
//
// All three are quadrature-free or per-point-cheap: bytes dominate for the
// Helmholtz load (HBM-bound), FP64 for the residuals.  Layout: one thread per cell
// (Burgers: per (cell, component); warp = component, lane = cell), the CTA's inputs
// staged once into shared memory by a coalesced copy of its contiguous cell range
// (odd row strides: conflict-free per-lane rows), reference tables read through the
// read-only path (every lane of a warp reads the same entry: one broadcast), and the
// element vectors staged back for a coalesced (or +=) store of the contiguous
// output range.
#include "common.cuh"
#include "femgpu_internal.h"
#include "../../include/femgpu.h"

namespace femgpu {

namespace {

constexpr int VEC_THREADS = 128;

__device__ __forceinline__ double ldro(const double* p) { return __ldg(p); }

// coalesced copy of `rows` rows of `w` doubles (contiguous in global) into padded smem
// rows, as asynchronous copies (cp.async: every element of the CTA's range in flight at
// once, no register round trip); stage_wait() + __syncthreads() before use
__device__ __forceinline__ void stage_rows(double* s, int stride, const double* g, int rows, int w) {
  for (int i = threadIdx.x; i < rows * w; i += blockDim.x)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(&s[(i / w) * stride + i % w])),
                 "l"(g + i)
                 : "memory");
}
__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void store_rows(double* g, const double* s, int stride, int rows, int w,
                                           int acc) {
  for (int i = threadIdx.x; i < rows * w; i += blockDim.x) {
    const double v = s[(i / w) * stride + i % w];
    if (acc)
      g[i] += v;
    else
      g[i] = v;
  }
}
constexpr int odd(int x) { return x % 2 ? x : x + 1; }

// ---------------------------------------------------------------------------
// Helmholtz load: b_j = |det| sum_m M_jm f_m, as one FP64 tensor-core GEMM per CTA:
// [128 cells x NC] (f, staged) x [NC x NS] (M^T, fragments held in registers for the
// whole kernel) on mma.sync m16n8k4 (DMMA); the epilogue scales row e by |det_e|.
// A thread-per-cell loop would issue one broadcast load of M per FMA (400 per cell
// for P3): load-issue bound at ~1.6 TB/s; the GEMM keeps the kernel on HBM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

template <int NS, int NC>
__global__ void __launch_bounds__(VEC_THREADS) vec_helm_kernel(long E, const double* __restrict__ coords,
                                                               const double* __restrict__ coef,
                                                               const double* __restrict__ M,
                                                               double* __restrict__ b, int acc) {
  constexpr int CELLS = VEC_THREADS, XS = 13, FS = odd(NC), OS = odd(NS);
  constexpr int KS = (NC + 3) / 4, NT = (NS + 7) / 8;  // k4 steps, n8 tiles
  constexpr int MT = CELLS / 16 / (VEC_THREADS / 32);   // m16 tiles per warp
  __shared__ double sx[CELLS * XS];
  __shared__ double sf[CELLS * (FS > OS ? FS : OS)];
  __shared__ double sdet[CELLS];
  const long c0 = (long)blockIdx.x * CELLS;
  const int nt = (int)min((long)CELLS, E - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  // B = M^T fragments: b[n][k] = M[8n + g][4k + t4] (zero padded)
  double bf[NT][KS];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int j = 8 * n + g, m = 4 * k + t4;
      bf[n][k] = (j < NS && m < NC) ? ldro(&M[j * NC + m]) : 0.0;
    }
  stage_rows(sx, XS, coords + c0 * 12, nt, 12);
  stage_rows(sf, FS, coef + c0 * NC, nt, NC);
  stage_wait();
  __syncthreads();
  {
    const int t = threadIdx.x;
    double x[12];
#pragma unroll
    for (int r = 0; r < 12; ++r) x[r] = t < nt ? sx[t * XS + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
    sdet[t] = cell_geometry(x).adet;
  }
  double cf[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r0 = (warp * MT + mt) * 16 + g;  // rows r0 and r0 + 8 of the CTA's cells
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int v = 0; v < 4; ++v) cf[mt][n][v] = 0.0;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const int m = 4 * k + t4;
      const double a0 = (m < NC && r0 < nt) ? sf[r0 * FS + m] : 0.0;
      const double a1 = (m < NC && r0 + 8 < nt) ? sf[(r0 + 8) * FS + m] : 0.0;
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma_16x8x4(cf[mt][n], a0, a1, bf[n][k]);
    }
  }
  __syncthreads();  // sf is reused as the output staging; sdet complete
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int r0 = (warp * MT + mt) * 16 + g;
    const double d0 = sdet[r0], d1 = sdet[r0 + 8];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int row = r0 + 8 * (v >> 1), j = 8 * n + 2 * t4 + (v & 1);
        if (j < NS) sf[row * OS + j] = (v >> 1 ? d1 : d0) * cf[mt][n][v];
      }
  }
  __syncthreads();
  store_rows(b + c0 * NS, sf, OS, nt, NS, acc);
}

// ---------------------------------------------------------------------------
// St Venant-Kirchhoff residual, vector P_k (NS scalar dofs per component)
// tab: W[Q] | D[3][Q][NS] | P[Q][4];  coeffs: w (3 x NS) | mu(4) | lam(4)
// ---------------------------------------------------------------------------
#ifndef VEC_SVK_MINB
#define VEC_SVK_MINB 2  // CTAs per SM the SVK residual kernel is register-capped for
#endif
#ifndef VEC_SVK_MUNROLL
#define VEC_SVK_MUNROLL 10  // unroll of its per-point gradient loop over the dofs
#endif
constexpr int kSvkMUnroll = VEC_SVK_MUNROLL;
template <int NS>
__global__ void __launch_bounds__(VEC_THREADS, VEC_SVK_MINB) vec_svk_kernel(long E, int Q,
                                                              const double* __restrict__ coords,
                                                              const double* __restrict__ coef,
                                                              const double* __restrict__ tab,
                                                              double* __restrict__ r, int acc) {
  constexpr int CELLS = VEC_THREADS, NCOEF = 3 * NS + 8, N = 3 * NS;
  constexpr int XS = 13, CS = odd(NCOEF), OS = odd(N);
  static_assert(OS <= CS + XS, "output staging fits the input rows");
  extern __shared__ __align__(16) double vsm[];
  double* sx = vsm;                  // [CELLS][XS]
  double* sc = vsm + CELLS * XS;     // [CELLS][CS]
  const double* W = tab;
  const double* D = tab + Q;
  const double* P = D + 3 * Q * NS;
  const long c0 = (long)blockIdx.x * CELLS;
  const int nt = (int)min((long)CELLS, E - c0);
  stage_rows(sx, XS, coords + c0 * 12, nt, 12);
  stage_rows(sc, CS, coef + c0 * NCOEF, nt, NCOEF);
  stage_wait();
  __syncthreads();
  const int t = threadIdx.x;
  double rc[3][NS];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int j = 0; j < NS; ++j) rc[c][j] = 0.0;
  if (t < nt) {
    double x[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) x[i] = sx[t * XS + i];
    const Geo g = cell_geometry(x);
    const double* w = sc + t * CS;
#pragma unroll 1
    for (int q = 0; q < Q; ++q) {
      double muq = 0.0, lamq = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double p = ldro(&P[q * 4 + m]);
        muq = fma(w[3 * NS + m], p, muq);
        lamq = fma(w[3 * NS + 4 + m], p, lamq);
      }
      // reference gradients of w: gr[c][a] = sum_m w_cm D_a,qm
      double gr[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll(kSvkMUnroll)
      for (int m = 0; m < NS; ++m) {
        double d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) d[a] = ldro(&D[(a * Q + q) * NS + m]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double wm = w[c * NS + m];
#pragma unroll
          for (int a = 0; a < 3; ++a) gr[c][a] = fma(wm, d[a], gr[c][a]);
        }
      }
      double F[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int bb = 0; bb < 3; ++bb)
          F[c][bb] = (c == bb ? 1.0 : 0.0) + gr[c][0] * g.K[0][bb] + gr[c][1] * g.K[1][bb] +
                     gr[c][2] * g.K[2][bb];
      double Ee[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          const double s = F[0][a] * F[0][bb] + F[1][a] * F[1][bb] + F[2][a] * F[2][bb];
          Ee[a][bb] = 0.5 * (a == bb ? s - 1.0 : s);
        }
      const double trE = Ee[0][0] + Ee[1][1] + Ee[2][2];
      const double wq = ldro(&W[q]) * g.adet;
      // T = wq (F S) K^T
      double FS[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          double s = 0.0;
#pragma unroll
          for (int p = 0; p < 3; ++p)
            s = fma(F[c][p], (p == bb ? lamq * trE : 0.0) + 2.0 * muq * Ee[p][bb], s);
          FS[c][bb] = wq * s;
        }
      double T[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          T[c][a] = FS[c][0] * g.K[a][0] + FS[c][1] * g.K[a][1] + FS[c][2] * g.K[a][2];
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        double d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) d[a] = ldro(&D[(a * Q + q) * NS + j]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          rc[c][j] = fma(T[c][0], d[0], fma(T[c][1], d[1], fma(T[c][2], d[2], rc[c][j])));
      }
    }
  }
  __syncthreads();  // the input rows are reused as the output staging
  if (t < nt) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int j = 0; j < NS; ++j) vsm[t * OS + c * NS + j] = rc[c][j];
  }
  __syncthreads();
  store_rows(r + c0 * N, vsm, OS, nt, N, acc);
}

// ---------------------------------------------------------------------------
// Burgers residual, vector P3: two FP64 tensor-core GEMMs per 16-cell tile and chunk
// of BZQ = 6 quadrature points (the quadrature schedule of sharing.cpp:409-607 with
// its two contractions on DMMA).  Rows = (component c, cell): m16 tile c.
//   A:  V[(c,e)][(q,s)] = sum_m u_{e,c,m} T_s[q][m]      T_0 = B, T_{1+a} = D_a
//       -> u_c(q), reference gradient of u_c at q             (K = 20, N = 6 x 4)
//   B:  per (cell, q), in place: adv_c = wq (u_c/dt + u . grad u_c),
//       t_ca = wq nu sum_b K_ab (grad u_c)_b,  wq = W_q |det|
//   C:  r[(c,e)][j] += sum_(q,s) Y[(c,e)][(q,s)] T_s[q][j]    (K = 6 x 4, N = 20 -> 24)
// 3 warps: phase A warp w computes n-tile w (2 points x 4 tables) of all 3 m-tiles
// (the u fragments of the tile live in registers); phase B one thread per (cell,
// point); phase C warp w owns component w's 3 output n-tiles for the whole tile.
// tab: W[Qp] | T[4][Qp][NS] (Qp = Q rounded up to BZQ, zero rows past Q).
// ---------------------------------------------------------------------------
constexpr int BZQ = 6;
constexpr int bz_qpad(int Q) { return (Q + BZQ - 1) / BZQ * BZQ; }

template <int NS>
__global__ void __launch_bounds__(96) vec_burgers_kernel(long E, int Q, const double* __restrict__ coords,
                                                         const double* __restrict__ coef,
                                                         const double* __restrict__ tab, double nu,
                                                         double dt, double* __restrict__ r, int acc) {
  constexpr int CELLS = 16, NCOEF = 3 * NS, N = 3 * NS;
  constexpr int XS = 13, CS = odd(NCOEF), OS = odd(N);
  constexpr int KA = (NS + 3) / 4, NTJ = (NS + 7) / 8;  // GEMM-A k4 steps; GEMM-C n8 tiles
  constexpr int VS = 4 * BZQ + 1;                        // V/Y row stride (odd)
  static_assert(NS % 4 == 0, "u fragments: whole k4 steps");
  __shared__ double sx[CELLS * XS];
  __shared__ double sc[CELLS * (CS > OS ? CS : OS)];
  __shared__ double sV[3 * CELLS * VS];
  __shared__ double sK[CELLS * 10];
  const int Qp = bz_qpad(Q);
  const double* W = tab;
  const double* T = tab + Qp;  // [4][Qp][NS]
  const long c0 = (long)blockIdx.x * CELLS;
  const int nt = (int)min((long)CELLS, E - c0);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, t4 = lane & 3;
  stage_rows(sx, XS, coords + c0 * 12, nt, 12);
  stage_rows(sc, CS, coef + c0 * NCOEF, nt, NCOEF);
  stage_wait();
  __syncthreads();
  if (tid < CELLS) {
    double x[12];
#pragma unroll
    for (int i = 0; i < 12; ++i)  // cells past the end: reference tet (never stored)
      x[i] = tid < nt ? sx[tid * XS + i] : ((i == 3 || i == 7 || i == 11) ? 1.0 : 0.0);
    const Geo geo = cell_geometry(x);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) sK[tid * 10 + a * 3 + b] = geo.K[a][b];
    sK[tid * 10 + 9] = geo.adet;
  }
  // GEMM-A A fragments: u_{cell, c, m}, m-tile c, rows g / g+8, k = 4k + t4
  double ua[3][KA][2];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const int m = 4 * k + t4;
      ua[c][k][0] = g < nt ? sc[g * CS + c * NS + m] : 0.0;
      ua[c][k][1] = g + 8 < nt ? sc[(g + 8) * CS + c * NS + m] : 0.0;
    }
  double racc[NTJ][4];
#pragma unroll
  for (int n = 0; n < NTJ; ++n)
#pragma unroll
    for (int v = 0; v < 4; ++v) racc[n][v] = 0.0;
  const double rdt = 1.0 / dt;
  __syncthreads();  // sK ready
#pragma unroll 1
  for (int q0 = 0; q0 < Qp; q0 += BZQ) {
    // ---- phase A: warp w -> columns 8w .. 8w+7 = (points q0 + 2w + {0,1}) x (tables 0..3)
    {
      double cv[3][4];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int v = 0; v < 4; ++v) cv[c][v] = 0.0;
      const int ql = 2 * w + (g >> 2), sb = g & 3;  // this lane's B column (point, table)
      const double* Tb = T + ((size_t)sb * Qp + q0 + ql) * NS;
#pragma unroll
      for (int k = 0; k < KA; ++k) {
        const double bfr = ldro(&Tb[4 * k + t4]);
#pragma unroll
        for (int c = 0; c < 3; ++c) dmma_16x8x4(cv[c], ua[c][k][0], ua[c][k][1], bfr);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          sV[(c * CELLS + g + 8 * (v >> 1)) * VS + 8 * w + 2 * t4 + (v & 1)] = cv[c][v];
    }
    __syncthreads();
    // ---- phase B: thread -> (cell, point), in place V -> Y
    {
      const int e = tid / BZQ, ql = tid % BZQ;
      const double* Kc = sK + e * 10;
      double uq[3], gu[3][3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double* v = sV + (c * CELLS + e) * VS + 4 * ql;
        uq[c] = v[0];
#pragma unroll
        for (int b = 0; b < 3; ++b) gu[c][b] = Kc[0 * 3 + b] * v[1] + Kc[1 * 3 + b] * v[2] + Kc[2 * 3 + b] * v[3];
      }
      const double wq = ldro(&W[q0 + ql]) * Kc[9];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double* y = sV + (c * CELLS + e) * VS + 4 * ql;
        y[0] = wq * (uq[c] * rdt + uq[0] * gu[c][0] + uq[1] * gu[c][1] + uq[2] * gu[c][2]);
#pragma unroll
        for (int a = 0; a < 3; ++a)
          y[1 + a] = wq * nu * (Kc[a * 3 + 0] * gu[c][0] + Kc[a * 3 + 1] * gu[c][1] + Kc[a * 3 + 2] * gu[c][2]);
      }
    }
    __syncthreads();
    // ---- phase C: warp w = component; k4 step kk = point q0 + kk, k = table t4
    {
      const double* y = sV + (w * CELLS) * VS;
#pragma unroll
      for (int kk = 0; kk < BZQ; ++kk) {
        const double a0 = y[g * VS + 4 * kk + t4], a1 = y[(g + 8) * VS + 4 * kk + t4];
        const double* Tc = T + ((size_t)t4 * Qp + q0 + kk) * NS;
#pragma unroll
        for (int n = 0; n < NTJ; ++n) {
          const int j = 8 * n + g;
          dmma_16x8x4(racc[n], a0, a1, j < NS ? ldro(&Tc[j]) : 0.0);
        }
      }
    }
    __syncthreads();  // Y consumed before the next chunk's phase A overwrites it
  }
  // element vectors: rows g / g+8 = cells, columns j = 8n + 2 t4 (+1), component w
#pragma unroll
  for (int n = 0; n < NTJ; ++n)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int cell = g + 8 * (v >> 1), j = 8 * n + 2 * t4 + (v & 1);
      if (j < NS) sc[cell * OS + w * NS + j] = racc[n][v];
    }
  __syncthreads();
  store_rows(r + c0 * N, sc, OS, nt, N, acc);
}

template <int NS, int NC>
cudaError_t launch_helm_t(long E, const double* x, const double* f, const double* M, double* b,
                          int acc, cudaStream_t s) {
  const long grid = (E + VEC_THREADS - 1) / VEC_THREADS;
  vec_helm_kernel<NS, NC><<<(unsigned)grid, VEC_THREADS, 0, s>>>(E, x, f, M, b, acc);
  return cudaGetLastError();
}

}  // namespace

int vector_table_qpad(int nq) { return bz_qpad(nq); }

bool vector_supported(int kind, int ns, int nc) {
  switch (kind) {
    case FEMGPU_HELMHOLTZ:
      return (ns == nc && (ns == 4 || ns == 10 || ns == 20)) || (nc == 4 && (ns == 10 || ns == 20));
    case FEMGPU_HYPERELASTICITY:
      return ns == 10 && nc == 4;
    case FEMGPU_BURGERS:
      return ns == 20;
    default:
      return false;
  }
}

cudaError_t launch_vector(int kind, int nq, int ns, int nc, long E, const double* coords,
                          const double* coef, const double* tab, const double* consts, double* out,
                          int acc, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  if (E > 0x7fffffffL * 32L) return cudaErrorInvalidValue;
  switch (kind) {
    case FEMGPU_HELMHOLTZ:
      if (ns == 4 && nc == 4) return launch_helm_t<4, 4>(E, coords, coef, tab, out, acc, s);
      if (ns == 10 && nc == 10) return launch_helm_t<10, 10>(E, coords, coef, tab, out, acc, s);
      if (ns == 20 && nc == 20) return launch_helm_t<20, 20>(E, coords, coef, tab, out, acc, s);
      if (ns == 10 && nc == 4) return launch_helm_t<10, 4>(E, coords, coef, tab, out, acc, s);
      if (ns == 20 && nc == 4) return launch_helm_t<20, 4>(E, coords, coef, tab, out, acc, s);
      break;
    case FEMGPU_HYPERELASTICITY:
      if (ns == 10) {
        constexpr size_t smem = sizeof(double) * VEC_THREADS * (13 + odd(3 * 10 + 8));
        static const char once_key = 0;  // one per (kernel instantiation, device)
        const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
          return cudaFuncSetAttribute(vec_svk_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem);
        });
        if (e0 != cudaSuccess) return e0;
        const long grid = (E + VEC_THREADS - 1) / VEC_THREADS;
        vec_svk_kernel<10><<<(unsigned)grid, VEC_THREADS, smem, s>>>(E, nq, coords, coef, tab, out, acc);
        return cudaGetLastError();
      }
      break;
    case FEMGPU_BURGERS:
      if (ns == 20) {
        const long grid = (E + 15) / 16;
        vec_burgers_kernel<20><<<(unsigned)grid, 96, 0, s>>>(E, nq, coords, coef, tab, consts[0],
                                                              consts[1], out, acc);
        return cudaGetLastError();
      }
      break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
