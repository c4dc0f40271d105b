// burgers.cu -- Burgers Jacobian element kernel, vector P3 (BASELINE config 5).
//
//   a(du,v) = int du.v/dt + (du.grad)u.v + (u.grad)du.v + nu grad du:grad v
//   A_{(c,j),(d,k)} = M^{cd}_{jk} + delta_cd C_{jk}
//   M^{cd}_{jk} = int phi_j phi_k d_d u_c         (symmetric in j,k)
//   C_{jk}      = int phi_j (u.grad phi_k) + nu grad phi_j.grad phi_k + phi_j phi_k / dt
//
// femopt cannot optimize the monolithic IR (exact cover limit, sharing.cpp:355,
// SURVEY.md App. A P5); per component block it pre-evaluates part of the
// monomials (P14: ~0.91 M flops/cell).  Here the whole Jacobian is a TENSOR
// schedule (pre-evaluation, preeval.cpp:279-451) factored into two FP64
// tensor-core GEMMs per 16-cell tile (mma.sync m16n8k4 f64 -> DMMA):
//
//  GEMM-1 (per component c):  H^{c,a}_{jk} = sum_n u_{c,n} T^{n,a}_{jk}
//         T^{n,a}_{jk} = sum_q W D_a(phi_n) phi_j phi_k  (resident in smem)
//         M^{cd}_{jk} = |det| sum_a K_ad H^{c,a}_{jk}   (reference -> physical)
//  GEMM-2 (once):             C_{jk} = sum_alpha g_alpha R_{alpha,jk}
//         alpha = (n,a): |det| sum_b u_{b,n} K_ab  x  sum_q W phi_n phi_j D_a(phi_k)
//                 s:     |det| nu (K K^T)_s       x  sum_q W D_a phi_j D_b phi_k (+ sym)
//                 mass:  |det| / dt               x  sum_q W phi_j phi_k
//         (B fragments streamed from L2 straight into registers)
//
// Output layout without staging: the 20x20 (j,k) plane is cut into 4x4
// blocks; a warp owns whole upper blocks (J<=K).  An n8 fragment covers two
// block rows, so every lane holds a 16-byte row segment and lane pairs form
// full 32-byte sectors of A_e.  The mirror block (K,J) reuses the same
// registers (M is symmetric); its C part comes from GEMM-2 columns permuted so
// that C_{kj} lands in the lane that writes position (k,j).  No shuffles, no
// shared-memory staging, no block-level synchronisation inside a tile.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

namespace bz {
constexpr int NS = 20;
constexpr int N = 60;
constexpr int NBU = 15;            // upper 4x4 blocks (J <= K) of the 20x20 (j,k) plane
constexpr int NT1 = 3 * NBU * 2;   // GEMM-1 n8 tiles: (a, upper block, half)
constexpr int KS1 = 5;             // GEMM-1 k4 steps (n = 0..19)
constexpr int KS2 = 17;            // GEMM-2 k4 steps: 60 (n,a) + 6 (G) + 1 (mass) + pad
constexpr int NT2 = 50;            // GEMM-2 n8 tiles: 15 direct + 10 mirror blocks, x2 halves
constexpr int CELLS = 16;
constexpr int THREADS = 256;
constexpr int WARPS = 8;
constexpr int T1_DBL = KS1 * NT1 * 32;         // 14400
constexpr int R2_DBL = KS2 * NT2 * 32;         // 27200
constexpr int A1_DBL = 3 * KS1 * 64;           // u_c fragments
constexpr int A2_DBL = KS2 * 64;               // g2 fragments
constexpr int IN_DBL = CELLS * (12 + 3 * NS);  // coords | u (cp.async target)
constexpr int CELLD = 10;                      // K(9), adet
constexpr size_t SMEM =
    sizeof(double) * (size_t)(T1_DBL + A1_DBL + A2_DBL + IN_DBL + CELLS * CELLD);
}  // namespace bz

// Upper block u (row-major over J <= K) -> (J, K).
__host__ __device__ constexpr int bz_J(int u) {
  return u < 5 ? 0 : u < 9 ? 1 : u < 12 ? 2 : u < 14 ? 3 : 4;
}
__host__ __device__ constexpr int bz_K(int u) {
  return u < 5 ? u : u < 9 ? u - 4 : u < 12 ? u - 7 : u < 14 ? u - 9 : 4;
}
// Off-diagonal upper blocks in order get GEMM-2 mirror slots 0..9.
__host__ __device__ constexpr int bz_mirror_slot(int u) {
  return bz_J(u) == bz_K(u) ? -1 : u - (bz_J(u) + 1);
}

// Warp work lists (upper blocks), balanced for GEMM-1 + GEMM-2 cost per SM
// sub-partition (warps w and w+4 share one).
__constant__ int c_wblk[bz::WARPS][2] = {{0, 5}, {1, 9}, {2, 12}, {3, 14}, {4, 6},
                                         {7, 8}, {10, 11}, {13, -1}};

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

__device__ __forceinline__ void cp_async8b(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void stg64(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

__global__ void __launch_bounds__(256, 1)
    burgers_kernel(long E, const double* __restrict__ coords, const double* __restrict__ u,
                   const double* __restrict__ tab, double nu, double dt,
                   double* __restrict__ A, int acc) {
  using namespace bz;
  extern __shared__ __align__(16) double smem[];
  double* sT1 = smem;                   // [KS1][NT1][32]  (m16n8k4 B fragments)
  double* sA1 = sT1 + T1_DBL;           // [3][KS1][32][2]
  double* sA2 = sA1 + A1_DBL;           // [KS2][32][2]
  double* sIn = sA2 + A2_DBL;           // [CELLS][12] | [CELLS][60]
  double* sCell = sIn + IN_DBL;         // [CELLS][10]
  const double* gR2 = tab + T1_DBL;     // [KS2][NT2][32]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  for (int i = tid; i < T1_DBL / 2; i += THREADS)
    reinterpret_cast<double2*>(sT1)[i] = reinterpret_cast<const double2*>(tab)[i];

  const long ntiles = (E + CELLS - 1) / CELLS;
  auto prefetch = [&](long tile) {
    const long c0 = tile * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    for (int i = tid; i < nt * 12; i += THREADS) cp_async8b(&sIn[i], coords + c0 * 12 + i);
    for (int i = tid; i < nt * 3 * NS; i += THREADS)
      cp_async8b(&sIn[CELLS * 12 + i], u + c0 * 3 * NS + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if ((long)blockIdx.x < ntiles) prefetch(blockIdx.x);

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = tile * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();  // inputs landed; previous tile's readers of sA1/sA2/sCell done
    if (tid < CELLS) {
      double x[12];
#pragma unroll
      for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
        x[r] = tid < nt ? sIn[tid * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
      const Geo geo = cell_geometry(x);
      double* cd = sCell + tid * CELLD;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) cd[a * 3 + b] = geo.K[a][b];
      cd[9] = geo.adet;
    }
    __syncthreads();
    // ---- A fragments: u_c (GEMM-1) and g2 (GEMM-2); a[v] = A[g + 8v][t] ----
    for (int i = tid; i < 3 * KS1 * 64; i += THREADS) {
      const int c = i / (KS1 * 64), r = i % (KS1 * 64);
      const int ks = r / 64, ln = (r % 64) / 2, v = r % 2;
      const int cell = (ln >> 2) + 8 * v, n = ks * 4 + (ln & 3);
      sA1[i] = cell < nt ? sIn[CELLS * 12 + cell * 3 * NS + c * NS + n] : 0.0;
    }
    for (int i = tid; i < KS2 * 64; i += THREADS) {
      const int ks = i / 64, ln = (i % 64) / 2, v = i % 2;
      const int cell = (ln >> 2) + 8 * v, al = ks * 4 + (ln & 3);
      const double* cd = sCell + cell * CELLD;
      const double* uc = sIn + CELLS * 12 + cell * 3 * NS;
      double val = 0.0;
      if (cell < nt) {
        if (al < 60) {
          const int n = al / 3, a = al % 3;  // beta_{n,a} = sum_b u_{b,n} K_ab
          val = cd[9] * (uc[n] * cd[a * 3 + 0] + uc[NS + n] * cd[a * 3 + 1] +
                         uc[2 * NS + n] * cd[a * 3 + 2]);
        } else if (al < 66) {
          const int s = al - 60;  // (0,0),(1,1),(2,2),(0,1),(0,2),(1,2)
          const int a = s < 3 ? s : (s == 5 ? 1 : 0);
          const int b = s < 3 ? s : (s == 3 ? 1 : 2);
          val = cd[9] * nu *
                (cd[a * 3 + 0] * cd[b * 3 + 0] + cd[a * 3 + 1] * cd[b * 3 + 1] +
                 cd[a * 3 + 2] * cd[b * 3 + 2]);
        } else if (al == 66) {
          val = cd[9] / dt;
        }
      }
      sA2[i] = val;
    }
    __syncthreads();
    if (tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);

    // per-lane cell data for rows g and g+8
    double Kc[2][9], ad[2];
#pragma unroll
    for (int vh = 0; vh < 2; ++vh) {
      const double* cd = sCell + (g + 8 * vh) * CELLD;
#pragma unroll
      for (int i = 0; i < 9; ++i) Kc[vh][i] = cd[i];
      ad[vh] = cd[9];
    }
    const bool row_ok0 = g < nt, row_ok1 = g + 8 < nt;

#pragma unroll 1
    for (int wb = 0; wb < 2; ++wb) {
      const int ub = c_wblk[warp][wb];
      if (ub < 0) break;
      const int J = bz_J(ub), K = bz_K(ub);
      const int ms = bz_mirror_slot(ub);
      const bool mirror = ms >= 0;
      // ---- GEMM-2: C direct (tiles 2ub, 2ub+1) and mirror (30 + 2ms + h) ----
      double cdir[2][4], cmir[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 4; ++v) cdir[h][v] = cmir[h][v] = 0.0;
      {
        const int td = 2 * ub, tm = 30 + 2 * (mirror ? ms : 0);
        double b0[4] = {0, 0, 0, 0}, b1[4] = {0, 0, 0, 0};
        auto loadB = [&](int ks, double (&b)[4]) {
          if (ks >= KS2) return;
          const double* base = gR2 + (size_t)ks * NT2 * 32 + lane;
          b[0] = ldg_nc(base + (td + 0) * 32);
          b[1] = ldg_nc(base + (td + 1) * 32);
          if (mirror) {
            b[2] = ldg_nc(base + (tm + 0) * 32);
            b[3] = ldg_nc(base + (tm + 1) * 32);
          }
        };
        auto step = [&](int ks, const double (&b)[4]) {
          const double2 a = reinterpret_cast<const double2*>(sA2)[ks * 32 + lane];
          dmma16x8x4(cdir[0], a.x, a.y, b[0]);
          dmma16x8x4(cdir[1], a.x, a.y, b[1]);
          if (mirror) {
            dmma16x8x4(cmir[0], a.x, a.y, b[2]);
            dmma16x8x4(cmir[1], a.x, a.y, b[3]);
          }
        };
        loadB(0, b0);
#pragma unroll 1
        for (int ks = 0; ks < KS2; ks += 2) {
          loadB(ks + 1, b1);
          step(ks, b0);
          if (ks + 1 < KS2) {
            loadB(ks + 2, b0);
            step(ks + 1, b1);
          }
        }
      }
      // ---- GEMM-1 per component c, then direct + mirror stores ------------
      // (unrolled: the delta_cd selection of C is resolved at compile time)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double hacc[3][2][4];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int v = 0; v < 4; ++v) hacc[a][h][v] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) {
          const double2 af = reinterpret_cast<const double2*>(sA1)[(c * KS1 + ks) * 32 + lane];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              dmma16x8x4(hacc[a][h], af.x, af.y,
                         sT1[(ks * NT1 + (a * NBU + ub) * 2 + h) * 32 + lane]);
        }
        // positions: row (cell g + 8vh), column pair e = 0,1 of tile h:
        //   jj = 2h + t/2, kk = 2(t%2) + e
#pragma unroll
        for (int vh = 0; vh < 2; ++vh) {
          if (!(vh ? row_ok1 : row_ok0)) continue;
          double* Ae = A + (c0 + g + 8 * vh) * (size_t)N * N;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 4 * J + 2 * h + (t >> 1);
            const int k = 4 * K + 2 * (t & 1);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              double m[2];
#pragma unroll
              for (int e = 0; e < 2; ++e)
                m[e] = ad[vh] * (Kc[vh][0 * 3 + d] * hacc[0][h][2 * vh + e] +
                                 Kc[vh][1 * 3 + d] * hacc[1][h][2 * vh + e] +
                                 Kc[vh][2 * 3 + d] * hacc[2][h][2 * vh + e]);
              const bool dg = (c == d);
              // direct: row (c, j), columns (d, k..k+1) -- 16 B, lane pairs fill a sector
              double2 vd = make_double2(m[0] + (dg ? cdir[h][2 * vh] : 0.0),
                                        m[1] + (dg ? cdir[h][2 * vh + 1] : 0.0));
              double2* pd = reinterpret_cast<double2*>(Ae + (c * NS + j) * N + d * NS + k);
              if (acc) {
                const double2 o = *pd;
                vd.x += o.x;
                vd.y += o.y;
              }
              stg_stream(pd, vd);
              if (mirror) {
                // mirror: rows (c, k+e), column (d, j); C part = C_{k+e, j}
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  double* pm = Ae + (c * NS + k + e) * N + d * NS + j;
                  double vm = m[e] + (dg ? cmir[h][2 * vh + e] : 0.0);
                  if (acc) vm += *pm;
                  stg64(pm, vm);
                }
              }
            }
          }
        }
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
  // column (upper block ub, half h, col) -> (j, k): jj = 2h + col/4, kk = col%4
  auto jk_of = [&](int ub, int h, int col, int* j, int* k) {
    *j = 4 * bz_J(ub) + 2 * h + col / 4;
    *k = 4 * bz_K(ub) + col % 4;
  };
  // T[n][a][j][k] (symmetric in j,k)
  static thread_local double T[NS][3][NS][NS];
  for (int n = 0; n < NS; ++n)
    for (int a = 0; a < 3; ++a)
      for (int j = 0; j < NS; ++j)
        for (int k = j; k < NS; ++k) {
          double s = 0.0;
          for (int q = 0; q < Q; ++q) s += W[q] * Dv(a, q, n) * Bv(q, j) * Bv(q, k);
          T[n][a][j][k] = T[n][a][k][j] = s;
        }
  for (int ks = 0; ks < KS1; ++ks)
    for (int a = 0; a < 3; ++a)
      for (int ub = 0; ub < NBU; ++ub)
        for (int h = 0; h < 2; ++h)
          for (int lane = 0; lane < 32; ++lane) {
            const int g = lane >> 2, t = lane & 3;
            const int n = ks * 4 + t;
            int j, k;
            jk_of(ub, h, g, &j, &k);
            out[((size_t)ks * NT1 + (a * NBU + ub) * 2 + h) * 32 + lane] =
                n < NS ? T[n][a][j][k] : 0.0;
          }
  // R2[alpha][j][k]
  static thread_local double R2[KS2 * 4][NS][NS];
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
            const int sI = al - 60;
            const int a = sI < 3 ? sI : (sI == 5 ? 1 : 0);
            const int b = sI < 3 ? sI : (sI == 3 ? 1 : 2);
            v = Dv(a, q, j) * Dv(b, q, k);
            if (a != b) v += Dv(b, q, j) * Dv(a, q, k);
          } else if (al == 66) {
            v = Bv(q, j) * Bv(q, k);
          }
          s += W[q] * v;
        }
        R2[al][j][k] = s;
      }
  double* r2 = out + T1_DBL;
  for (int ub = 0; ub < NBU; ++ub) {
    const int ms = bz_mirror_slot(ub);
    for (int h = 0; h < 2; ++h)
      for (int ks = 0; ks < KS2; ++ks)
        for (int lane = 0; lane < 32; ++lane) {
          const int g = lane >> 2, t = lane & 3;
          int j, k;
          jk_of(ub, h, g, &j, &k);
          const int al = ks * 4 + t;
          // direct tile: C[j][k]
          r2[((size_t)ks * NT2 + 2 * ub + h) * 32 + lane] = R2[al][j][k];
          // mirror tile: the lane that writes position (k, j) needs C[k][j]
          if (ms >= 0) r2[((size_t)ks * NT2 + 30 + 2 * ms + h) * 32 + lane] = R2[al][k][j];
        }
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
