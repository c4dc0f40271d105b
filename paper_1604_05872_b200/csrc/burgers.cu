// burgers.cu -- Burgers Jacobian element kernel, vector P3 (BASELINE config 5).
//
//   a(du,v) = int du.v/dt + (du.grad)u.v + (u.grad)du.v + nu grad du:grad v
//   A_{(c,j),(d,k)} = M^{cd}_{jk} + delta_cd C_{jk}
//   M^{cd}_{jk} = int phi_j phi_k d_d u_c         (symmetric in j,k)
//   C_{jk}      = int phi_j (u.grad phi_k) + nu grad phi_j.grad phi_k + phi_j phi_k / dt
//
// femopt cannot optimize the monolithic IR (exact cover limit, sharing.cpp:355,
// SURVEY.md App. A P5) and per component block it pre-evaluates only part of
// the monomials (P14, ~0.91 M flops/cell).  Here the whole Jacobian is a
// TENSOR schedule (pre-evaluation, preeval.cpp:279-451) factored so the
// per-cell work is two FP64 tensor-core GEMMs (mma.sync m16n8k4 f64 -> DMMA):
//
//  GEMM-1 (per component c):  H^{c,a}_p = sum_n u_{c,n} T^{n,a}_p
//         T^{n,a}_{jk} = sum_q W D_a(phi_n) phi_j phi_k   (20 x 3*210, resident in smem)
//         then M^{cd}_p = |det| sum_a K_ad H^{c,a}_p   (reference->physical, epilogue)
//  GEMM-2 (once):             C_jk = sum_alpha g_alpha R_alpha,jk
//         alpha = (n,a): |det| sum_b u_{b,n} K_ab  x  sum_q W phi_n phi_j D_a(phi_k)
//                 s:     |det| nu (K K^T)_s       x  sum_q W D_a phi_j D_b phi_k (+ sym)
//                 mass:  |det| / dt               x  sum_q W phi_j phi_k
//         (68 x 400, B fragments streamed straight from L2 into registers)
//
// Per 16-cell tile: ~66 k FMA/cell on the tensor cores.  Output slabs (rows
// (c, j), all 60 columns: 9.6 KB contiguous per cell and c) are staged through
// shared memory four cells at a time and stored with coalesced 16-byte writes.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

namespace bz {
constexpr int NS = 20;
constexpr int N = 60;
constexpr int NP = 210;            // j <= k pairs
constexpr int PPAD = 216;          // p columns per a-slice (27 n8 tiles)
constexpr int PT = 27;             // p-tiles per a-slice
constexpr int NT1 = 3 * PT;        // GEMM-1 n8 tiles (a, p)
constexpr int KS1 = 5;             // GEMM-1 k4 steps (n = 0..19)
constexpr int KR2 = 67;            // GEMM-2 real K: 60 (n,a) + 6 (G) + 1 (mass)
constexpr int KS2 = 17;            // GEMM-2 k4 steps (68)
constexpr int NT2 = 50;            // GEMM-2 n8 tiles (400 columns)
constexpr int CELLS = 16;
constexpr int THREADS = 256;
constexpr int OUTC = 4;            // cells per staging round
constexpr int T1_DBL = KS1 * NT1 * 32;        // 12960
constexpr int R2_DBL = KS2 * NT2 * 32;        // 27200
constexpr int A1_DBL = 3 * KS1 * 64;          // u_c fragments
constexpr int A2_DBL = KS2 * 64;              // g2 fragments
constexpr int IN_DBL = CELLS * (12 + 3 * NS);  // coords | u
constexpr int CELLD = 10;                     // K(9), adet
constexpr int C_DBL = CELLS * NS * NS;        // C tile
constexpr int STG_DBL = OUTC * NS * N;        // 4 slabs of 20 x 60
constexpr size_t SMEM = sizeof(double) * (size_t)(T1_DBL + C_DBL + STG_DBL + A1_DBL + A2_DBL +
                                                  IN_DBL + CELLS * CELLD) +
                        sizeof(int) * NP;
}  // namespace bz

__device__ __forceinline__ void dmma16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ double ldg_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(256, 1)
    burgers_kernel(long E, const double* __restrict__ coords, const double* __restrict__ u,
                   const double* __restrict__ tab, double nu, double dt,
                   double* __restrict__ A, int acc) {
  using namespace bz;
  extern __shared__ __align__(16) double smem[];
  double* sT1 = smem;                   // [KS1][NT1][32]  (m16n8k4 B fragments)
  double* sC = sT1 + T1_DBL;            // [CELLS][20][20]
  double* sStg = sC + C_DBL;            // [OUTC][20][60]
  double* sA1 = sStg + STG_DBL;         // [3][KS1][32][2]
  double* sA2 = sA1 + A1_DBL;           // [KS2][32][2]
  double* sIn = sA2 + A2_DBL;           // [CELLS][12] | [CELLS][60]
  double* sCell = sIn + IN_DBL;         // [CELLS][10]
  int* sPair = reinterpret_cast<int*>(sCell + CELLS * CELLD);
  const double* gR2 = tab + T1_DBL;     // [KS2][NT2][32]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  for (int i = tid; i < T1_DBL / 2; i += THREADS)
    reinterpret_cast<double2*>(sT1)[i] = reinterpret_cast<const double2*>(tab)[i];
  for (int j = 0, p = 0; j < NS; ++j)
    for (int k = j; k < NS; ++k, ++p)
      if (p % THREADS == tid) sPair[p] = (j << 8) | k;

  // GEMM-2 n-tiles of this warp: 7,7,6,6,6,6,6,6
  const int nt2_begin = warp * 6 + min(warp, 2);
  const int nt2_count = 6 + (warp < 2 ? 1 : 0);

  const long ntiles = (E + CELLS - 1) / CELLS;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = tile * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    __syncthreads();
    // ---- inputs ----------------------------------------------------------
    for (int i = tid; i < CELLS * 12; i += THREADS) {
      const int c = i / 12, r = i % 12;
      const double ref = (r == 3 || r == 7 || r == 11) ? 1.0 : 0.0;
      sIn[i] = c < nt ? coords[(c0 + c) * 12 + r] : ref;
    }
    for (int i = tid; i < CELLS * 3 * NS; i += THREADS) {
      const int c = i / (3 * NS);
      sIn[CELLS * 12 + i] = c < nt ? u[c0 * 3 * NS + i] : 0.0;
    }
    __syncthreads();
    if (tid < CELLS) {
      const Geo geo = cell_geometry(&sIn[tid * 12]);
      double* cd = sCell + tid * CELLD;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) cd[a * 3 + b] = geo.K[a][b];
      cd[9] = geo.adet;
    }
    __syncthreads();
    // ---- A fragments: u_c (GEMM-1) and g2 (GEMM-2) ------------------------
    // m16n8k4 A fragment: a[v] = A[row g + 8v][col t]
    for (int i = tid; i < 3 * KS1 * 64; i += THREADS) {
      const int c = i / (KS1 * 64), r = i % (KS1 * 64);
      const int ks = r / 64, ln = (r % 64) / 2, v = r % 2;
      const int cell = (ln >> 2) + 8 * v, n = ks * 4 + (ln & 3);
      sA1[i] = n < NS ? sIn[CELLS * 12 + cell * 3 * NS + c * NS + n] : 0.0;
    }
    for (int i = tid; i < KS2 * 64; i += THREADS) {
      const int ks = i / 64, ln = (i % 64) / 2, v = i % 2;
      const int cell = (ln >> 2) + 8 * v, al = ks * 4 + (ln & 3);
      const double* cd = sCell + cell * CELLD;
      const double* uc = sIn + CELLS * 12 + cell * 3 * NS;
      double val = 0.0;
      if (al < 60) {
        const int n = al / 3, a = al % 3;  // beta_{n,a} = sum_b u_{b,n} K_ab
        val = cd[9] * (uc[n] * cd[a * 3 + 0] + uc[NS + n] * cd[a * 3 + 1] +
                       uc[2 * NS + n] * cd[a * 3 + 2]);
      } else if (al < 66) {
        const int s = al - 60;
        // s: (0,0),(1,1),(2,2),(0,1),(0,2),(1,2)
        const int a = s < 3 ? s : (s == 5 ? 1 : 0);
        const int b = s < 3 ? s : (s == 3 ? 1 : 2);
        val = cd[9] * nu *
              (cd[a * 3 + 0] * cd[b * 3 + 0] + cd[a * 3 + 1] * cd[b * 3 + 1] +
               cd[a * 3 + 2] * cd[b * 3 + 2]);
      } else if (al == 66) {
        val = cd[9] / dt;
      }
      sA2[i] = val;
    }
    __syncthreads();

    // ---- GEMM-2: C[16 cells][400] ------------------------------------------
    {
      double c2[7][4];
#pragma unroll
      for (int i = 0; i < 7; ++i) c2[i][0] = c2[i][1] = c2[i][2] = c2[i][3] = 0.0;
      double b0[7], b1[7];
      auto loadB = [&](int ks, double (&b)[7]) {
#pragma unroll
        for (int i = 0; i < 7; ++i)
          b[i] = (i < nt2_count && ks < KS2)
                     ? ldg_nc(gR2 + ((size_t)ks * NT2 + nt2_begin + i) * 32 + lane)
                     : 0.0;
      };
      auto mma_step = [&](int ks, const double (&b)[7]) {
        const double2 a = reinterpret_cast<const double2*>(sA2)[ks * 32 + lane];
#pragma unroll
        for (int i = 0; i < 7; ++i)
          if (i < nt2_count) dmma16x8x4(c2[i], a.x, a.y, b[i]);
      };
      // register double buffer, prefetch distance 1 (B from L2, no smem staging:
      // each fragment feeds exactly one warp)
      loadB(0, b0);
#pragma unroll 1
      for (int ks = 0; ks < KS2; ks += 2) {
        loadB(ks + 1, b1);
        mma_step(ks, b0);
        if (ks + 1 < KS2) {
          loadB(ks + 2, b0);
          mma_step(ks + 1, b1);
        }
      }
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        if (i >= nt2_count) break;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int cell = g + 8 * (v >> 1);
          const int col = (nt2_begin + i) * 8 + 2 * t + (v & 1);
          sC[cell * NS * NS + col] = c2[i][v];
        }
      }
    }
    __syncthreads();

    // ---- GEMM-1 per component c, epilogue per 4-cell round ------------------
#pragma unroll 1
    for (int c = 0; c < 3; ++c) {
      double h[4][3][4];  // [p-tile][a][frag]
      double af[KS1][2];
#pragma unroll
      for (int ks = 0; ks < KS1; ++ks) {
        const double2 a = reinterpret_cast<const double2*>(sA1)[(c * KS1 + ks) * 32 + lane];
        af[ks][0] = a.x;
        af[ks][1] = a.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int pt = warp + 8 * i;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          h[i][a][0] = h[i][a][1] = h[i][a][2] = h[i][a][3] = 0.0;
          if (pt < PT) {
#pragma unroll
            for (int ks = 0; ks < KS1; ++ks)
              dmma16x8x4(h[i][a], af[ks][0], af[ks][1], sT1[(ks * NT1 + a * PT + pt) * 32 + lane]);
          }
        }
      }
#pragma unroll 1
      for (int r = 0; r < CELLS / OUTC; ++r) {
        const int vh = r >> 1;                 // fragment half holding these cells
        const int gl = (r & 1) * 4;            // g range [gl, gl+4)
        if (g >= gl && g < gl + 4) {
          const int cell = g + 8 * vh;
          const int lc = cell - r * OUTC;
          const double* cd = sCell + cell * CELLD;
          double* slab = sStg + lc * NS * N;
          const double* Cc = sC + cell * NS * NS;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int pt = warp + 8 * i;
            if (pt >= PT) break;
#pragma unroll
            for (int vv = 0; vv < 2; ++vv) {
              const int p = pt * 8 + 2 * t + vv;
              if (p >= NP) continue;
              // register select (no dynamic indexing of the fragment arrays)
              const double h0 = vh ? h[i][0][2 + vv] : h[i][0][vv];
              const double h1 = vh ? h[i][1][2 + vv] : h[i][1][vv];
              const double h2 = vh ? h[i][2][2 + vv] : h[i][2][vv];
              const int jk = sPair[p];
              const int j = jk >> 8, k = jk & 0xff;
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                const double m = cd[9] * (cd[0 * 3 + d] * h0 + cd[1 * 3 + d] * h1 + cd[2 * 3 + d] * h2);
                const bool diag = (d == c);
                slab[j * N + d * NS + k] = m + (diag ? Cc[j * NS + k] : 0.0);
                if (j != k) slab[k * N + d * NS + j] = m + (diag ? Cc[k * NS + j] : 0.0);
              }
            }
          }
        }
        __syncthreads();
        const long cb = c0 + r * OUTC;
        const int ncell = (int)max(0L, min((long)OUTC, E - cb));
        for (int i = tid; i < ncell * NS * N / 2; i += THREADS) {
          const int lc = i / (NS * N / 2), w = i % (NS * N / 2);
          double2 v = reinterpret_cast<const double2*>(sStg)[i];
          double2* dst = reinterpret_cast<double2*>(A + (cb + lc) * (size_t)N * N + c * NS * N) + w;
          if (acc) {
            const double2 o = *dst;
            v.x += o.x;
            v.y += o.y;
          }
          stg_stream(dst, v);
        }
        __syncthreads();
      }
    }
  }
}

bool burgers_supported(int nq, int ns) { return ns == bz::NS && nq > 0; }

void burgers_tables(int nq, const double* W, const double* B, const double* D, double* out) {
  // out = [T1 fragments (KS1*NT1*32) | R2 fragments (KS2*NT2*32)]
  using namespace bz;
  const int Q = nq;
  auto Bv = [&](int q, int j) { return B[(size_t)q * NS + j]; };
  auto Dv = [&](int a, int q, int j) { return D[((size_t)a * Q + q) * NS + j]; };
  // T[n][a][p]
  static thread_local double T[NS][3][NP];
  for (int n = 0; n < NS; ++n)
    for (int a = 0; a < 3; ++a) {
      int p = 0;
      for (int j = 0; j < NS; ++j)
        for (int k = j; k < NS; ++k, ++p) {
          double s = 0.0;
          for (int q = 0; q < Q; ++q) s += W[q] * Dv(a, q, n) * Bv(q, j) * Bv(q, k);
          T[n][a][p] = s;
        }
    }
  for (int ks = 0; ks < KS1; ++ks)
    for (int nt = 0; nt < NT1; ++nt)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        const int n = ks * 4 + t, col = nt * 8 + g, a = col / PPAD, p = col % PPAD;
        out[((size_t)ks * NT1 + nt) * 32 + lane] = (n < NS && p < NP) ? T[n][a][p] : 0.0;
      }
  // R2[alpha][jk]
  static thread_local double R2[KS2 * 4][NS * NS];
  const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
  for (int al = 0; al < KS2 * 4; ++al)
    for (int j = 0; j < NS; ++j)
      for (int k = 0; k < NS; ++k) {
        double s = 0.0;
        for (int q = 0; q < Q; ++q) {
          double v = 0.0;
          if (al < 60) {
            const int n = al / 3, a = al % 3;
            v = Bv(q, n) * Bv(q, j) * Dv(a, q, k);
          } else if (al < 66) {
            const int a = ab[al - 60][0], b = ab[al - 60][1];
            v = Dv(a, q, j) * Dv(b, q, k);
            if (a != b) v += Dv(b, q, j) * Dv(a, q, k);
          } else if (al == 66) {
            v = Bv(q, j) * Bv(q, k);
          }
          s += W[q] * v;
        }
        R2[al][j * NS + k] = s;
      }
  double* r2 = out + T1_DBL;
  for (int ks = 0; ks < KS2; ++ks)
    for (int nt = 0; nt < NT2; ++nt)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        r2[((size_t)ks * NT2 + nt) * 32 + lane] = R2[ks * 4 + t][nt * 8 + g];
      }
}

size_t burgers_table_doubles() { return bz::T1_DBL + bz::R2_DBL; }

cudaError_t launch_burgers(int ns, long E, const double* coords, const double* coef,
                           const double* tab, double nu, double dt, double* A, int acc,
                           cudaStream_t s) {
  if (ns != bz::NS) return cudaErrorInvalidValue;
  if (E <= 0) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(burgers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bz::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const long ntiles = (E + bz::CELLS - 1) / bz::CELLS;
  const int grid = (int)(ntiles < kNumSMs ? ntiles : kNumSMs);
  burgers_kernel<<<grid, bz::THREADS, bz::SMEM, s>>>(E, coords, coef, tab, nu, dt, A, acc);
  return cudaGetLastError();
}

}  // namespace femgpu
