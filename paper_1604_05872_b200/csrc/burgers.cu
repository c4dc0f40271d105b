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
//         (B fragments through a 4-deep TMA bulk-copy ring, mbarrier full/empty)
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
constexpr int KS2 = 18;            // GEMM-2 k4 steps: 60 (n,a) + 6 (G) + 1 (mass) + pad
constexpr int KPS2 = 3;            // k4 steps per ring stage
constexpr int NST2 = KS2 / KPS2;   // ring stages per pass
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
// GEMM-2 B operand: TMA ring of per-k-step stages.  A tile runs two passes (the
// first and second block of every warp); pass p's stage holds only the n8
// tiles its warps need (30 resp. 20), laid out contiguously on the host.
constexpr int NB = 3;                          // ring depth
constexpr int SLOTS0 = 30, SLOTS1 = 20;
constexpr int STAGE_MAX = KPS2 * SLOTS0 * 32;  // doubles
constexpr int R2_OFF1 = KS2 * SLOTS0 * 32;     // pass-1 offset inside the R2 table
constexpr size_t SMEM = sizeof(double) * (size_t)(T1_DBL + A1_DBL + A2_DBL + IN_DBL +
                                                  CELLS * CELLD + NB * STAGE_MAX) +
                        2 * NB * sizeof(uint64_t);
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
// sub-partition (warps w and w+4 share one).  Warp 7 (one block only) doubles
// as the TMA producer of the GEMM-2 ring.
constexpr int kWblk[bz::WARPS][2] = {{0, 5}, {1, 9}, {2, 12}, {3, 14}, {4, 6},
                                     {7, 8}, {10, 11}, {13, -1}};
__constant__ int c_wblk[bz::WARPS][2] = {{0, 5}, {1, 9}, {2, 12}, {3, 14}, {4, 6},
                                         {7, 8}, {10, 11}, {13, -1}};
// first GEMM-2 slot of warp w in pass p (direct h0, h1, then mirror h0, h1)
constexpr int bz_slot_base(int w, int p) {
  int off = 0;
  for (int x = 0; x < w; ++x) {
    const int ub = kWblk[x][p];
    if (ub >= 0) off += (bz_J(ub) == bz_K(ub)) ? 2 : 4;
  }
  return off;
}
__constant__ int c_slot[bz::WARPS][2] = {
    {bz_slot_base(0, 0), bz_slot_base(0, 1)}, {bz_slot_base(1, 0), bz_slot_base(1, 1)},
    {bz_slot_base(2, 0), bz_slot_base(2, 1)}, {bz_slot_base(3, 0), bz_slot_base(3, 1)},
    {bz_slot_base(4, 0), bz_slot_base(4, 1)}, {bz_slot_base(5, 0), bz_slot_base(5, 1)},
    {bz_slot_base(6, 0), bz_slot_base(6, 1)}, {bz_slot_base(7, 0), bz_slot_base(7, 1)}};
static_assert(bz_slot_base(bz::WARPS, 0) == bz::SLOTS0, "pass-0 slot count");
static_assert(bz_slot_base(bz::WARPS, 1) == bz::SLOTS1, "pass-1 slot count");

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

__device__ __forceinline__ void mbar_arrive_cta_bz(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
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
  double* sRing = sCell + CELLS * CELLD;  // [NB][STAGE_MAX]  GEMM-2 B stages
  uint64_t* rFull = reinterpret_cast<uint64_t*>(sRing + NB * STAGE_MAX);
  uint64_t* rEmpty = rFull + NB;
  const double* gR2 = tab + T1_DBL;     // [pass][KS2][slots][32]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;

  for (int i = tid; i < T1_DBL / 2; i += THREADS)
    reinterpret_cast<double2*>(sT1)[i] = reinterpret_cast<const double2*>(tab)[i];

  const long ntiles = (E + CELLS - 1) / CELLS;
  const long my_tiles =
      (long)blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const long total_stages = my_tiles * 2 * NST2;
  const bool producer = (warp == WARPS - 1) && lane == 0;
  auto issue_stage = [&](long gs) {  // stage gs -> ring slot gs % NB
    const int b = (int)(gs % NB);
    const int pass = (int)((gs / NST2) & 1), st = (int)(gs % NST2);
    const int slots = pass ? SLOTS1 : SLOTS0;
    const double* src = gR2 + (pass ? R2_OFF1 : 0) + (size_t)st * KPS2 * slots * 32;
    mbar_expect_tx(&rFull[b], KPS2 * slots * 32 * 8);
    bulk_g2s(sRing + b * STAGE_MAX, src, KPS2 * slots * 32 * 8, &rFull[b]);
  };
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) {
      mbar_init(&rFull[b], 1);
      mbar_init(&rEmpty[b], WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (producer)
    for (long gs = 0; gs < NB && gs < total_stages; ++gs) issue_stage(gs);
  // consume stage gs (wait full), release it, and (producer) refill the slot
  auto stage_wait = [&](long gs) {
    mbar_wait(&rFull[gs % NB], (uint32_t)((gs / NB) & 1));
  };
  auto stage_release = [&](long gs) {
    __syncwarp();
    if (lane == 0) mbar_arrive_cta_bz(&rEmpty[gs % NB]);
    if (producer && gs + NB < total_stages) {
      mbar_wait(&rEmpty[gs % NB], (uint32_t)((gs / NB) & 1));
      issue_stage(gs + NB);
    }
  };
  long it = -1;
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
    ++it;
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
      const long gs0 = (it * 2 + wb) * NST2;  // first ring stage of this pass
      if (ub < 0) {  // no block in this pass: keep the ring moving
#pragma unroll 1
        for (int st = 0; st < NST2; ++st) {
          stage_wait(gs0 + st);
          stage_release(gs0 + st);
        }
        continue;
      }
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
        const int slot = c_slot[warp][wb];
        const int slots = wb ? SLOTS1 : SLOTS0;
#pragma unroll 1
        for (int st = 0; st < NST2; ++st) {
          const long gs = gs0 + st;
          stage_wait(gs);
          const double* stb = sRing + (gs % NB) * STAGE_MAX + slot * 32 + lane;
          double bq[KPS2][4];
          double2 aq[KPS2];
#pragma unroll
          for (int kk = 0; kk < KPS2; ++kk) {  // all operand loads of the stage first
            const double* p = stb + kk * slots * 32;
            bq[kk][0] = p[0];
            bq[kk][1] = p[32];
            bq[kk][2] = mirror ? p[64] : 0.0;
            bq[kk][3] = mirror ? p[96] : 0.0;
            aq[kk] = reinterpret_cast<const double2*>(sA2)[(st * KPS2 + kk) * 32 + lane];
          }
          stage_release(gs);
#pragma unroll
          for (int kk = 0; kk < KPS2; ++kk) {
            dmma16x8x4(cdir[0], aq[kk].x, aq[kk].y, bq[kk][0]);
            dmma16x8x4(cdir[1], aq[kk].x, aq[kk].y, bq[kk][1]);
            if (mirror) {
              dmma16x8x4(cmir[0], aq[kk].x, aq[kk].y, bq[kk][2]);
              dmma16x8x4(cmir[1], aq[kk].x, aq[kk].y, bq[kk][3]);
            }
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
          const bool ok = vh ? row_ok1 : row_ok0;  // lane-pair uniform (same g)
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
              if (ok) {
                if (acc) {
                  const double2 o = *pd;
                  vd.x += o.x;
                  vd.y += o.y;
                }
                stg_stream(pd, vd);
              }
              if (mirror) {
                // mirror: rows (c, k+e), column (d, j); C part = C_{k+e, j}.  Lanes
                // t and t^2 hold columns j, j+1 of rows k, k+1: swap one value so
                // each lane stores a 16-byte row segment.
                const double vm0 = m[0] + (dg ? cmir[h][2 * vh] : 0.0);
                const double vm1 = m[1] + (dg ? cmir[h][2 * vh + 1] : 0.0);
                const bool lo = (t >> 1) == 0;
                const double other = __shfl_xor_sync(0xffffffffu, lo ? vm1 : vm0, 2);
                const int jj0 = 4 * J + 2 * h;  // even column of the pair
                double2* pm = reinterpret_cast<double2*>(
                    Ae + (c * NS + k + (lo ? 0 : 1)) * N + d * NS + jj0);
                double2 vmv = lo ? make_double2(vm0, other) : make_double2(other, vm1);
                if (ok) {
                  if (acc) {
                    const double2 o = *pm;
                    vmv.x += o.x;
                    vmv.y += o.y;
                  }
                  stg_stream(pm, vmv);
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
  // [pass][ks][slot][32]: warp w's slots of pass p start at bz_slot_base(w, p)
  double* r2 = out + T1_DBL;
  for (int p = 0; p < 2; ++p) {
    const int slots = p ? SLOTS1 : SLOTS0;
    double* base = r2 + (p ? R2_OFF1 : 0);
    for (int w = 0; w < WARPS; ++w) {
      const int ub = kWblk[w][p];
      if (ub < 0) continue;
      const bool off = bz_J(ub) != bz_K(ub);
      const int s0 = bz_slot_base(w, p);
      for (int h = 0; h < 2; ++h)
        for (int ks = 0; ks < KS2; ++ks)
          for (int lane = 0; lane < 32; ++lane) {
            const int g = lane >> 2, t = lane & 3;
            int j, k;
            jk_of(ub, h, g, &j, &k);
            const int al = ks * 4 + t;
            // direct tile: C[j][k]
            base[((size_t)ks * slots + s0 + h) * 32 + lane] = R2[al][j][k];
            // mirror tile: the lane that writes position (k, j) needs C[k][j]
            if (off) base[((size_t)ks * slots + s0 + 2 + h) * 32 + lane] = R2[al][k][j];
          }
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
