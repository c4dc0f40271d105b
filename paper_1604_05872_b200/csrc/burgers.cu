// burgers.cu -- Burgers Jacobian element kernel, vector P3 (BASELINE config 5).
//
//   a(du,v) = int du.v/dt + (du.grad)u.v + (u.grad)du.v + nu grad du:grad v
//   A_{(c,j),(d,k)} = M^{cd}_{jk} + delta_cd C_{jk}
//   M^{cd}_{jk} = int phi_j phi_k d_d u_c         (symmetric in j,k)
//   C_{jk}      = int phi_j (u.grad phi_k) + nu grad phi_j.grad phi_k + phi_j phi_k / dt
//
// femopt cannot optimize the monolithic IR (exact cover limit, sharing.cpp:355,
// SURVEY.md App. A P5); per component block it pre-evaluates part of the
// monomials (P14: ~0.91 M flops/cell).  Here the Jacobian is a TENSOR schedule
// (pre-evaluation, preeval.cpp:279-451) factored into two FP64 tensor-core
// GEMMs per 16-cell tile (mma.sync m16n8k4 f64 -> DMMA):
//
//  GEMM-1 (per (c,d)):  M^{cd}_{jk} = sum_m g^{cd}_m S_{m,jk}
//         The reference derivative tables D_a span the derivative space of
//         the element (P2 for P3: rank r = 10 <= 12) at the quadrature
//         points.  With an orthonormal basis Psi (Q x r) of that span,
//         D_a = Psi Dn_a exactly, so d_d u_c(x_q) = sum_m Psi_qm g^{cd}_m,
//         g^{cd}_m = |det| sum_a K_ad (Dn_a u_c)_m   (per cell, CUDA cores)
//         S_{m,jk}  = sum_q W_q Psi_qm phi_j(q) phi_k(q)   (host, once)
//  GEMM-2 (once):       C_{jk} = sum_alpha g_alpha R_{alpha,jk}
//         alpha = (n,a): |det| sum_b u_{b,n} K_ab  x  sum_q W phi_n phi_j D_a(phi_k)
//                 s:     |det| nu (K K^T)_s       x  sum_q W D_a phi_j D_b phi_k (+ sym)
//                 mass:  |det| / dt               x  sum_q W phi_j phi_k
//
// Work split: the 20x20 (j,k) plane is cut into 4x4 blocks; the 15 upper
// blocks (J <= K) belong to warps 0..14 of a 16-warp CTA (one CTA per SM).
// Each warp keeps its block's S fragments in registers for the whole kernel,
// computes the block's C (direct + permuted mirror tiles, B fragments from L2)
// once per tile, then for each of the 9 (c,d) blocks of A_e: 6 DMMAs, + C on
// the diagonal, and writes the 4x4 block and its mirror into a shared-memory
// slab [16 cells][20][20].  Warp 15 issues one 3D TMA tensor store per slab
// (box 20 x 20 x 16 cells, clipped at E; cp.reduce...add for accumulate) and
// keeps up to two stores in flight, so HBM sees long, full-line write streams
// while the tensor cores work on the next block.  The element matrix (28.8 KB
// per cell) is written exactly once.
//
// Tile schedule (BZ_SCHED 1): the six off-diagonal (c,d) blocks need no C, so
// they go out first, through slabs 1 and 2, with GEMM-2's k4 steps in between
// (its B fragments stream through a 4-stage ring in slab 0) -- the store stream
// does not stop while C is built; then the three diagonal blocks (slabs 0, 1, 2).
// Measured 1.284 vs 1.314 ms (BZ_SCHED 0: GEMM-2 first over an 8-stage ring in
// slabs 0 and 1, then the nine blocks).  Ablations (BZ_ABL) show the kernel is
// not HBM-bound: without any TMA store 1.22 ms, without the slab writes 1.01 ms,
// without GEMM-2 1.13 ms -- the shared-memory crossbar (ring fill and reads,
// slab writes, the TMA's slab reads) and the DMMA pipe serialise per block.
// Stores straight from registers (16-byte, full sectors, no staging) ran 2.57 ms:
// 16 L2 transactions per warp instruction.  Staggering half the warps (GEMM-2
// chunk before the block, so slab writes and DMMA overlap) ran 2.01 ms; letting the
// last warp to write a slab issue its store (no designated issuer; atomics) 1.41 ms;
// a dedicated 17th issuer warp 1.43 ms (17 warps leave 96 registers per thread).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

#ifndef BZ_SCHED
#define BZ_SCHED 1  // 1: GEMM-2 interleaved with the off-diagonal blocks (ring in slab 0);
                    // 0: GEMM-2 first, then the nine blocks (ring in slabs 0 and 1)
#endif
#ifndef BZ_KFRONT
#define BZ_KFRONT 0  // BZ_SCHED 1: extra GEMM-2 k4 steps after the first off-diagonal block
#endif
#ifndef BZ_ABL  // development ablations (BZ_SCHED 1): 1 no TMA stores, 2 no GEMM-2,
                // 4 no GEMM-1 DMMA, 8 no slab writes
#define BZ_ABL 0
#endif
#ifndef BZ_RING_LA
#define BZ_RING_LA (BZ_SCHED ? 4 : 8)  // R2 stages in flight ahead of the consuming k4 step
#endif

namespace bz {
constexpr int NS = 20;
constexpr int N = 60;
constexpr int NBU = 15;            // upper 4x4 blocks (J <= K) of the 20x20 (j,k) plane
constexpr int KS1 = 3;             // GEMM-1 k4 steps over the derivative space
constexpr int RMAX = 4 * KS1;      // largest supported derivative-space rank
constexpr int DNR = 16;            // Dn rows held in smem (two n8 tiles, zero past rank)
constexpr int KS2 = 17;            // GEMM-2 k4 steps: 60 (n,a) + 6 (G) + 1 (mass) + 1 pad
constexpr int CELLS = 16;
constexpr int WARPS = 16;
constexpr int THREADS = 32 * WARPS;
constexpr int CWARPS = 15;         // compute warps, one upper block each
constexpr int CTHREADS = 32 * CWARPS;
constexpr int PRODUCER = 15;       // warp 15: inputs, geometry, GEMM A fragments
constexpr int ISSUER = 14;         // lane 0 of warp 14 issues the slab stores
constexpr int NSLAB = 3;
constexpr int SLAB_DBL = CELLS * NS * NS;     // one (c,d) block of 16 cells
constexpr int S_DBL = NBU * KS1 * 2 * 32;     // GEMM-1 B fragments
constexpr int R2_DBL = KS2 * 25 * 64;         // GEMM-2 B fragments [ks][pair][32][2]
constexpr int DN_DBL = 3 * DNR * NS;          // Dn_a (r x 20), zero rows past r
constexpr int A1_DBL = 9 * KS1 * 64;          // g^{cd} fragments
constexpr int A2_DBL = KS2 * 64;              // GEMM-2 A fragments
constexpr int COORD_DBL = CELLS * 12;
constexpr int IN_DBL = CELLS * (12 + 3 * NS); // coords | u (bulk-copy target)
constexpr int CELLD = 10;                     // K(9), adet
constexpr int NPAIR = 25;                     // GEMM-2 B tile pairs: 15 direct + 10 mirror
constexpr int STAGE_DBL = NPAIR * 64;         // one k4 step of R2
constexpr int NRING = BZ_SCHED ? 4 : 8;        // ring stages (alias slab 0, or slabs 0 and 1)
constexpr int RING_LA = BZ_RING_LA < NRING ? BZ_RING_LA : NRING;  // stages in flight
constexpr size_t SMEM =
    sizeof(double) * (size_t)(NSLAB * SLAB_DBL + DN_DBL + 2 * A1_DBL + 2 * A2_DBL + IN_DBL +
                              CELLS * CELLD) + 8 * (1 + 2 * 8 + 2 * 3);
static_assert(NRING * STAGE_DBL <= (BZ_SCHED ? 1 : 2) * SLAB_DBL, "R2 ring aliases slab 0 (and 1)");
// named barriers (0 = __syncthreads)
constexpr int BAR_CD = 1;          // compute warps, once per (c,d) block
constexpr int BAR_FULL = 2;        // + buffer: producer -> compute
constexpr int BAR_EMPTY = 4;       // + buffer: compute -> producer
}  // namespace bz

// Upper block u (row-major over J <= K) -> (J, K).
__host__ __device__ constexpr int bz_J(int u) {
  return u < 5 ? 0 : u < 9 ? 1 : u < 12 ? 2 : u < 14 ? 3 : 4;
}
__host__ __device__ constexpr int bz_K(int u) {
  return u < 5 ? u : u < 9 ? u - 4 : u < 12 ? u - 7 : u < 14 ? u - 9 : 4;
}

// Off-diagonal upper blocks in order -> 0..9 (their mirror GEMM-2 tile pair).
__host__ __device__ constexpr int bz_off_index(int u) {
  return u < 5 ? u - 1 : u < 9 ? u - 2 : u < 12 ? u - 3 : u < 14 ? u - 4 : -1;
}

// Warp -> upper block.  Sub-partition s runs warps s, s+4, s+8, s+12; the ten
// off-diagonal blocks (GEMM-2: 72 DMMA/tile) and five diagonal ones (36) are
// spread so that no sub-partition carries more than 3 off + 1 diagonal.
__constant__ int c_wblk[bz::WARPS] = {1, 2, 3, 4, 6, 7, 8, 10, 11, 13, 0, 5, 9, 12, 14, -1};

__device__ __forceinline__ void dmma16x8x4(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ double ldg_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ double2 ldg_nc2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void cp_async8b(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// The slabs are written once and never re-read: stores carry an L2 evict_first policy
// so they do not displace the R2 table and the streamed inputs (-2.2 % on c5; the
// same hint on the 1D bulk stores of pair.cu costs 0.3-1.2 %, so only here --
// profiles/c5_r02_ablation.txt).
#ifndef BZ_EVICT
#define BZ_EVICT 1
#endif
__device__ __forceinline__ void slab_store(const CUtensorMap* map, const double* src, int col,
                                           int row, int cell, int acc) {
  if (acc)
    asm volatile(
        "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group "
        "[%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
        "r"(col), "r"(row), "r"(cell), "r"(smem_u32(src))
        : "memory");
  else {
#if BZ_EVICT
    const uint64_t pol = l2_evict_first();
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint "
        "[%0, {%1, %2, %3}], [%4], %5;\n" ::"l"(map),
        "r"(col), "r"(row), "r"(cell), "r"(smem_u32(src)), "l"(pol)
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
            map),
        "r"(col), "r"(row), "r"(cell), "r"(smem_u32(src))
        : "memory");
#endif
  }
}

__device__ __forceinline__ void bulk_wait_read2() {
  asm volatile("cp.async.bulk.wait_group.read 2;\n" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void nbar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

#ifdef BZ_TRACE
// development trace (CTA 0 only): clock64 at pipeline milestones per tile
__device__ unsigned long long bz_trace[128][20];
#define BZ_MARK(it, slot, cond) \
  if (blockIdx.x == 0 && (cond) && (it) < 128) bz_trace[it][slot] = clock64()
#define BZ_T0() const unsigned long long bz_t0 = clock64()
#define BZ_ACC(it, slot) \
  if (blockIdx.x == 0 && (it) < 128) bz_trace[it][slot] += clock64() - bz_t0
extern "C" int femgpu_debug_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, bz_trace, sizeof(bz_trace));
}
#else
#define BZ_MARK(it, slot, cond)
#define BZ_T0()
#define BZ_ACC(it, slot)
#endif

__global__ void __launch_bounds__(bz::THREADS, 1)
    burgers_kernel(const __grid_constant__ CUtensorMap amap, long E,
                   const double* __restrict__ coords, const double* __restrict__ u,
                   const double* __restrict__ tab, double nu, double dt, int acc) {
  using namespace bz;
  extern __shared__ __align__(1024) double smem[];
  double* sSlab = smem;                    // [NSLAB][CELLS][20][20]  (TMA box layout)
  double* sDn = sSlab + NSLAB * SLAB_DBL;  // [3][DNR][20]
  double* sA1 = sDn + DN_DBL;              // [2][9][KS1][32][2]
  double* sA2 = sA1 + 2 * A1_DBL;          // [2][KS2][32][2]
  double* sIn = sA2 + 2 * A2_DBL;          // [CELLS][12] | [CELLS][60]
  double* sCell = sIn + IN_DBL;            // [CELLS][10]
  uint64_t* inBar = reinterpret_cast<uint64_t*>(sCell + CELLS * CELLD);
  uint64_t* rFull = inBar + 1;             // [NRING] R2 stage landed
  uint64_t* rEmpty = rFull + NRING;        // [NRING] R2 stage consumed by all compute warps
  double* sRing = sSlab;                   // [NRING][25][32][2]  (aliases slabs 0, 1)
  uint64_t* slabFull = rEmpty + NRING;     // [NSLAB] all compute threads wrote the block
  uint64_t* slabEmpty = slabFull + NSLAB;  // [NSLAB] the TMA unit has read the slab
  const double* gS = tab;                  // [ub][KS1][2][32]
  const double* gR2 = tab + S_DBL;         // [KS2][25][32][2]
  const double* gDn = gR2 + R2_DBL;        // [3][DNR][20]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long ntiles = (E + CELLS - 1) / CELLS;
  const long my_tiles =
      (long)blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  for (int i = tid; i < DN_DBL; i += THREADS) sDn[i] = gDn[i];
  if (tid == 0) {
    mbar_init(inBar, 1);
    for (int r = 0; r < NRING; ++r) {
      mbar_init(&rFull[r], 1);
      mbar_init(&rEmpty[r], CWARPS);
    }
    for (int r = 0; r < NSLAB; ++r) {
      mbar_init(&slabFull[r], CTHREADS);
      mbar_init(&slabEmpty[r], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == PRODUCER) {
    // ===================== producer: inputs -> A fragments =====================
    auto load = [&](long tile) {  // one bulk copy each for coords and u
      if (lane == 0) {
        const long c0 = tile * CELLS;
        const int nt = (int)min((long)CELLS, E - c0);
        mbar_expect_tx(inBar, nt * (12 + 3 * NS) * 8);
        bulk_g2s(sIn, coords + c0 * 12, nt * 12 * 8, inBar);
        bulk_g2s(sIn + COORD_DBL, u + c0 * 3 * NS, nt * 3 * NS * 8, inBar);
      }
    };
    if (my_tiles > 0) load(blockIdx.x);
    for (long it = 0; it < my_tiles; ++it) {
      const long tile = blockIdx.x + it * gridDim.x;
      const int nt = (int)min((long)CELLS, E - tile * CELLS);
      const int b = (int)(it & 1);
      double* A1 = sA1 + b * A1_DBL;
      double* A2 = sA2 + b * A2_DBL;
      mbar_wait(inBar, (uint32_t)(it & 1));
      BZ_MARK(it, 0, lane == 0);
      if (lane < CELLS) {
        double x[12];
#pragma unroll
        for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
          x[r] = lane < nt ? sIn[lane * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
        const Geo geo = cell_geometry(x);
        double* cd = sCell + lane * CELLD;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) cd[a * 3 + bb] = geo.K[a][bb];
        cd[9] = lane < nt ? geo.adet : 0.0;  // zero rows for cells past the end
      }
      if (it >= 2) nbar_sync(BAR_EMPTY + b, THREADS);  // compute warps done with buffer b
      BZ_MARK(it, 1, lane == 0);
      __syncwarp();
      // ---- GEMM-1 A: Gu_a = u_c Dn_a^T on the tensor cores (rows = cells,
      //      columns = m in two n8 tiles), then g^{cd}_m = |det| sum_a K_ad Gu_a ----
      const double* uin = sIn + COORD_DBL;
#pragma unroll 1
      for (int c = 0; c < 3; ++c) {
        double gu[3][2][4];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int tt = 0; tt < 2; ++tt)
#pragma unroll
            for (int v = 0; v < 4; ++v) gu[a][tt][v] = 0.0;
#pragma unroll
        for (int ks = 0; ks < NS / 4; ++ks) {
          const int n = ks * 4 + t;
          const double a0 = uin[g * 3 * NS + c * NS + n];
          const double a1 = uin[(g + 8) * 3 * NS + c * NS + n];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int tt = 0; tt < 2; ++tt)
              dmma16x8x4(gu[a][tt], a0, a1, sDn[(a * DNR + 8 * tt + g) * NS + n]);
        }
        // gu[a][tt][v] = Gu_a[cell g + 8(v>>1)][m = 8tt + 2t + (v&1)]
#pragma unroll
        for (int vh = 0; vh < 2; ++vh) {
          const int cell = g + 8 * vh;
          const double* cd = sCell + cell * CELLD;
          double Kd[3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int d = 0; d < 3; ++d) Kd[a][d] = cd[9] * cd[a * 3 + d];
#pragma unroll
          for (int tt = 0; tt < 2; ++tt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int m = 8 * tt + 2 * t + e;
              if (m < RMAX) {
                const int v = 2 * vh + e;
#pragma unroll
                for (int d = 0; d < 3; ++d)
                  A1[(((c * 3 + d) * KS1 + (m >> 2)) * 32 + 4 * (cell & 7) + (m & 3)) * 2 + vh] =
                      Kd[0][d] * gu[0][tt][v] + Kd[1][d] * gu[1][tt][v] + Kd[2][d] * gu[2][tt][v];
              }
            }
        }
      }
      BZ_MARK(it, 2, lane == 0);
      // ---- GEMM-2 A fragments a[v] = A[cell g + 8v][alpha = 4ks + t] ----
      {
        const int cell = lane & 15;
        const double* cd = sCell + cell * CELLD;
        double Kc[9];
        const double ad = cd[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) Kc[i] = cd[i];
        const double* uc = uin + cell * 3 * NS;
        auto put = [&](int al, double val) {
          A2[((al >> 2) * 32 + 4 * (cell & 7) + (al & 3)) * 2 + (cell >> 3)] = val;
        };
        // beta_{n,a} = |det| sum_b u_{b,n} K_ab at alpha = 3n + a
#pragma unroll 2
        for (int n = lane >> 4; n < NS; n += 2) {
          const double u0 = uc[n], u1 = uc[NS + n], u2 = uc[2 * NS + n];
#pragma unroll
          for (int a = 0; a < 3; ++a)
            put(3 * n + a, ad * (Kc[a * 3 + 0] * u0 + Kc[a * 3 + 1] * u1 + Kc[a * 3 + 2] * u2));
        }
        if (lane < 16) {  // nu |det| (K K^T)_s at 60..65, |det|/dt at 66, zero pad
#pragma unroll
          for (int s6 = 0; s6 < 6; ++s6) {
            const int a = s6 < 3 ? s6 : (s6 == 5 ? 1 : 0);
            const int bb = s6 < 3 ? s6 : (s6 == 3 ? 1 : 2);
            put(60 + s6, ad * nu *
                             (Kc[a * 3 + 0] * Kc[bb * 3 + 0] + Kc[a * 3 + 1] * Kc[bb * 3 + 1] +
                              Kc[a * 3 + 2] * Kc[bb * 3 + 2]));
          }
          put(66, ad / dt);
#pragma unroll
          for (int al = 67; al < 4 * KS2; ++al) put(al, 0.0);
        }
      }
      __syncwarp();
      // sIn fully consumed (reads retired into registers): refill with the next tile
      if (it + 1 < my_tiles) {
        fence_proxy_async();
        load(tile + gridDim.x);
      }
      BZ_MARK(it, 3, lane == 0);
      nbar_arrive(BAR_FULL + b, THREADS);
    }
    return;
  }

  // ======================= compute warps: one upper block each =================
  const int ub = c_wblk[warp];
  const int J = bz_J(ub), K = bz_K(ub);
  const bool mirror = J != K;
  const bool issuer = warp == ISSUER && lane == 0;  // slab stores + R2 ring refills
  const int hs = g & 1;  // odd-g lanes write the other half first (bank spread)
  // GEMM-1 B fragments of this warp's block: registers for the whole kernel
  double sb[KS1][2];
#pragma unroll
  for (int ks = 0; ks < KS1; ++ks)
#pragma unroll
    for (int h = 0; h < 2; ++h) sb[ks][h] = gS[((ub * KS1 + ks) * 2 + h) * 32 + lane];
#if BZ_SCHED
  // GEMM-2 B fragments stream through a ring of k4 stages [25 pairs][32][2]
  // aliasing slab 0 (BZ_SCHED 1) or slabs 0 and 1 (BZ_SCHED 0)
  const int pdir = ub, pmir = NBU + bz_off_index(ub);
  auto ring_issue = [&](long G) {  // stage G = tile * KS2 + ks -> slot G % NRING
    const int slot = (int)(G % NRING);
    const int ks = (int)(G % KS2);
    mbar_expect_tx(&rFull[slot], STAGE_DBL * 8);
    bulk_g2s(sRing + slot * STAGE_DBL, gR2 + (size_t)ks * STAGE_DBL, STAGE_DBL * 8, &rFull[slot]);
  };
  if (issuer && my_tiles > 0 && !(BZ_ABL & 2))
    for (int ks = 0; ks < RING_LA; ++ks) ring_issue(ks);

  double cdir[2][4], cmir[2][4];
  // one GEMM-2 k4 step of tile it: C direct (pair pdir) and mirror (pair pmir)
  auto gemm2_step = [&](long it, int ks, const double* A2, bool refill) {
    const long G = it * KS2 + ks;
    const int slot = (int)(G % NRING);
    mbar_wait(&rFull[slot], (uint32_t)((G / NRING) & 1));
    BZ_MARK(it, 16, tid == 0 && ks == 0);
    BZ_MARK(it, 19, tid == 0 && ks == KS2 - 1);
    const double2* st = reinterpret_cast<const double2*>(sRing + slot * STAGE_DBL);
    const double2 bd = st[pdir * 32 + lane];
    const double2 bm = mirror ? st[pmir * 32 + lane] : make_double2(0.0, 0.0);
    const double2 af = reinterpret_cast<const double2*>(A2)[ks * 32 + lane];
    __syncwarp();
    if (lane == 0) mbar_arrive1(&rEmpty[slot]);
    dmma16x8x4(cdir[0], af.x, af.y, bd.x);
    dmma16x8x4(cdir[1], af.x, af.y, bd.y);
    if (mirror) {
      dmma16x8x4(cmir[0], af.x, af.y, bm.x);
      dmma16x8x4(cmir[1], af.x, af.y, bm.y);
    }
    if (issuer && refill && ks + RING_LA < KS2) {  // stage ks + RING_LA into its slot
      const long G2 = G + RING_LA;
      if (G2 >= NRING) mbar_wait(&rEmpty[G2 % NRING], (uint32_t)(((G2 / NRING) - 1) & 1));
      ring_issue(G2);
    }
  };

  // one (c,d) block of tile it: GEMM-1, + C on the diagonal, written into the slab;
  // the issuer sends the slab with a TMA tensor store once every warp has written it
  int prev_slab = -1;  // issuer: slab of the previous store in flight
  // sl: slab, n: its use count (slab 0 once per tile, slabs 1 and 2 four times)
  auto block = [&](long it, long c0, int cdi, const double* A1, int sl, uint32_t n) {
    const int c = cdi / 3, d = cdi % 3;
    double* slab = sSlab + sl * SLAB_DBL;
    double m[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 4; ++v) m[h][v] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS1; ++ks) {
      const double2 af = reinterpret_cast<const double2*>(A1)[(cdi * KS1 + ks) * 32 + lane];
      if (BZ_ABL & 4) {
        m[0][ks] += af.x * sb[ks][0];
        m[1][ks] += af.y * sb[ks][1];
        continue;
      }
      dmma16x8x4(m[0], af.x, af.y, sb[ks][0]);
      dmma16x8x4(m[1], af.x, af.y, sb[ks][1]);
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {  // odd-g lanes: half 1 first
      const double m0 = m[0][v], m1 = m[1][v];
      m[0][v] = hs ? m1 : m0;
      m[1][v] = hs ? m0 : m1;
    }
    double r[2][4];  // mirror values
#pragma unroll
    for (int hi = 0; hi < 2; ++hi)
#pragma unroll
      for (int v = 0; v < 4; ++v) r[hi][v] = m[hi][v];
    if (c == d) {
#pragma unroll
      for (int hi = 0; hi < 2; ++hi)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          r[hi][v] += cmir[hi][v];
          m[hi][v] += cdir[hi][v];
        }
    }
    if (n > 0) mbar_wait(&slabEmpty[sl], (n - 1) & 1);
#pragma unroll
    for (int hi = 0; hi < 2 && !(BZ_ABL & 8); ++hi) {
      const int h = hi ^ hs;
      const int j = 4 * J + 2 * h + (t >> 1);
      const int k = 4 * K + 2 * (t & 1);
#pragma unroll
      for (int vh = 0; vh < 2; ++vh) {
        double* cellp = slab + (g + 8 * vh) * (NS * NS);
        *reinterpret_cast<double2*>(cellp + j * NS + k) =
            make_double2(m[hi][2 * vh], m[hi][2 * vh + 1]);
        if (mirror) {
          const bool lo = (t >> 1) == 0;
          const double other =
              __shfl_xor_sync(0xffffffffu, lo ? r[hi][2 * vh + 1] : r[hi][2 * vh], 2);
          const int jj0 = 4 * J + 2 * h;
          *reinterpret_cast<double2*>(cellp + (k + (lo ? 0 : 1)) * NS + jj0) =
              lo ? make_double2(r[hi][2 * vh], other) : make_double2(other, r[hi][2 * vh + 1]);
        }
      }
    }
    fence_proxy_async();  // generic-proxy slab writes -> visible to the TMA unit
    mbar_arrive1(&slabFull[sl]);
    if (issuer) {
      {
        BZ_T0();
        mbar_wait(&slabFull[sl], n & 1);
        BZ_ACC(it, 15);
      }
      if (!(BZ_ABL & 1)) slab_store(&amap, slab, d * NS, c * NS, (int)c0, acc);
      bulk_commit();
      if (prev_slab >= 0) {
        BZ_T0();
        bulk_wait_read1();  // the previous store has left its slab
        BZ_ACC(it, 18);
        mbar_arrive1(&slabEmpty[prev_slab]);
      }
      prev_slab = sl;
    }
  };
  auto swap_c = [&]() {  // odd-g lanes handle half 1 first: swap C once per tile
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double d0 = cdir[0][v], d1 = cdir[1][v], m0 = cmir[0][v], m1 = cmir[1][v];
      cdir[0][v] = hs ? d1 : d0;
      cdir[1][v] = hs ? d0 : d1;
      cmir[0][v] = hs ? m1 : m0;
      cmir[1][v] = hs ? m0 : m1;
    }
  };

  // Tile schedule: the six off-diagonal blocks (no C) go out first, through slabs
  // 1 and 2, with GEMM-2's k4 steps between them -- the TMA store stream never
  // drains while the tensor cores build C; then the three diagonal blocks (slabs
  // 0, 1, 2: slab 0 is free once GEMM-2 is done).  Once the first diagonal store
  // has left slab 0, the issuer refills the ring there for the next tile.
  for (long it = 0; it < my_tiles; ++it) {
    const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
    const int b = (int)(it & 1);
    const double* A1 = sA1 + b * A1_DBL;
    const double* A2 = sA2 + b * A2_DBL;
    nbar_sync(BAR_FULL + b, THREADS);
    BZ_MARK(it, 4, tid == 0);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 4; ++v) cdir[h][v] = cmir[h][v] = 0.0;
    int ks = 0;
#pragma unroll 1
    for (int ob = 0; ob < 6; ++ob) {
      // off-diagonal (c,d) = 01 02 10 12 20 21 -> cdi 1 2 3 5 6 7
      block(it, c0, ob + 1 + (ob >= 3), A1, 1 + (ob & 1), (uint32_t)(4 * it + (ob >> 1)));
      BZ_MARK(it, 6 + ob, tid == 0);
      // GEMM-2 k4 steps done by the end of this block's chunk: BZ_KFRONT steps with
      // the first block, the rest spread evenly over the six
      const int kend = BZ_KFRONT + ((ob + 1) * (KS2 - BZ_KFRONT) + 5) / 6;
#pragma unroll 1
      for (; ks < kend && !(BZ_ABL & 2); ++ks) gemm2_step(it, ks, A2, true);
    }
    BZ_MARK(it, 5, tid == 0);
    swap_c();
    nbar_sync(BAR_CD, CTHREADS);  // every warp's ring reads done before slab 0 is written
#pragma unroll 1
    for (int di = 0; di < 3; ++di) {
      block(it, c0, 4 * di, A1, di, (uint32_t)(di == 0 ? it : 4 * it + 3));
      BZ_MARK(it, 12 + di, tid == 0);
      if (issuer && di == 1 && it + 1 < my_tiles && !(BZ_ABL & 2)) {
        // the first diagonal store (slab 0) has been read (wait_read1 in block):
        // the next tile's first ring stages into slab 0
        BZ_MARK(it, 17, true);
        for (int k = 0; k < RING_LA; ++k) {
          const long G = (it + 1) * KS2 + k;
          if (G >= NRING) mbar_wait(&rEmpty[G % NRING], (uint32_t)(((G / NRING) - 1) & 1));
          ring_issue(G);
        }
      }
    }
    if (it + 2 < my_tiles) nbar_arrive(BAR_EMPTY + b, THREADS);
  }
#else
  // GEMM-2 B fragments stream through a ring of k4 stages [25 pairs][32][2]
  // aliasing slabs 0 and 1 (free while GEMM-2 runs: the last stores of a tile
  // use slabs 2, 1, 0 in that order and have been read by the time we refill)
  const int pdir = ub, pmir = NBU + bz_off_index(ub);
  auto ring_issue = [&](long G) {  // stage G = tile * KS2 + ks -> slot G % NRING
    const int slot = (int)(G % NRING);
    const int ks = (int)(G % KS2);
    mbar_expect_tx(&rFull[slot], STAGE_DBL * 8);
    bulk_g2s(sRing + slot * STAGE_DBL, gR2 + (size_t)ks * STAGE_DBL, STAGE_DBL * 8, &rFull[slot]);
  };
  if (issuer && my_tiles > 0)
    for (int ks = 0; ks < RING_LA; ++ks) ring_issue(ks);

  long gi = 0;  // running (c,d) block counter of this CTA: slab gi % NSLAB
  for (long it = 0; it < my_tiles; ++it) {
    const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
    const int b = (int)(it & 1);
    const double* A1 = sA1 + b * A1_DBL;
    const double* A2 = sA2 + b * A2_DBL;
    nbar_sync(BAR_FULL + b, THREADS);
    BZ_MARK(it, 4, tid == 0);

    // ---- GEMM-2: C direct (pair pdir) and mirror (pair pmir) ----------------
    double cdir[2][4], cmir[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int v = 0; v < 4; ++v) cdir[h][v] = cmir[h][v] = 0.0;
#pragma unroll 2
    for (int ks = 0; ks < KS2; ++ks) {
      const long G = it * KS2 + ks;
      const int slot = (int)(G % NRING);
      mbar_wait(&rFull[slot], (uint32_t)((G / NRING) & 1));
      BZ_MARK(it, 16, tid == 0 && ks == 0);
      BZ_MARK(it, 19, tid == 0 && ks == KS2 - 1);
      const double2* st = reinterpret_cast<const double2*>(sRing + slot * STAGE_DBL);
      const double2 bd = st[pdir * 32 + lane];
      const double2 bm = mirror ? st[pmir * 32 + lane] : make_double2(0.0, 0.0);
      const double2 af = reinterpret_cast<const double2*>(A2)[ks * 32 + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive1(&rEmpty[slot]);
      dmma16x8x4(cdir[0], af.x, af.y, bd.x);
      dmma16x8x4(cdir[1], af.x, af.y, bd.y);
      if (mirror) {
        dmma16x8x4(cmir[0], af.x, af.y, bm.x);
        dmma16x8x4(cmir[1], af.x, af.y, bm.y);
      }
      if (issuer && ks + RING_LA < KS2) {  // stage ks + RING_LA into its slot
        const long G2 = G + RING_LA;
        if (G2 >= NRING) mbar_wait(&rEmpty[G2 % NRING], (uint32_t)(((G2 / NRING) - 1) & 1));
        ring_issue(G2);
      }
    }
    BZ_MARK(it, 5, tid == 0);
    // odd-g lanes handle half 1 first: swap C once per tile
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double d0 = cdir[0][v], d1 = cdir[1][v], m0 = cmir[0][v], m1 = cmir[1][v];
      cdir[0][v] = hs ? d1 : d0;
      cdir[1][v] = hs ? d0 : d1;
      cmir[0][v] = hs ? m1 : m0;
      cmir[1][v] = hs ? m0 : m1;
    }
    nbar_sync(BAR_CD, CTHREADS);  // ring reads done before slab 0/1 writes

    // ---- the nine (c,d) blocks: GEMM-1, + C on the diagonal, slab, TMA ----
#pragma unroll 1
    for (int cdi = 0; cdi < 9; ++cdi, ++gi) {
      const int c = cdi / 3, d = cdi % 3;
      double* slab = sSlab + (gi % NSLAB) * SLAB_DBL;
      double m[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int v = 0; v < 4; ++v) m[h][v] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS1; ++ks) {
        const double2 af = reinterpret_cast<const double2*>(A1)[(cdi * KS1 + ks) * 32 + lane];
        dmma16x8x4(m[0], af.x, af.y, sb[ks][0]);
        dmma16x8x4(m[1], af.x, af.y, sb[ks][1]);
      }
      // odd-g lanes: half 1 first
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double m0 = m[0][v], m1 = m[1][v];
        m[0][v] = hs ? m1 : m0;
        m[1][v] = hs ? m0 : m1;
      }
      double r[2][4];  // mirror values
#pragma unroll
      for (int hi = 0; hi < 2; ++hi)
#pragma unroll
        for (int v = 0; v < 4; ++v) r[hi][v] = m[hi][v];
      if (c == d) {
#pragma unroll
        for (int hi = 0; hi < 2; ++hi)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            r[hi][v] += cmir[hi][v];
            m[hi][v] += cdir[hi][v];
          }
      }
      if (gi >= NSLAB) mbar_wait(&slabEmpty[gi % NSLAB], (uint32_t)(((gi / NSLAB) - 1) & 1));
      // C fragment c[v] = C[cell g + 8(v>>1)][col 2t + (v&1)];
      // col -> (j, k) = (4J + 2h + t/2, 4K + 2(t&1) + e)
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        const int h = hi ^ hs;
        const int j = 4 * J + 2 * h + (t >> 1);
        const int k = 4 * K + 2 * (t & 1);
#pragma unroll
        for (int vh = 0; vh < 2; ++vh) {
          double* cellp = slab + (g + 8 * vh) * (NS * NS);
          *reinterpret_cast<double2*>(cellp + j * NS + k) =
              make_double2(m[hi][2 * vh], m[hi][2 * vh + 1]);
          if (mirror) {
            // mirror: rows k+e, column j.  Lanes t and t^2 hold columns j, j+1
            // of rows k, k+1: swap one value so each lane writes 16 bytes.
            const bool lo = (t >> 1) == 0;
            const double other =
                __shfl_xor_sync(0xffffffffu, lo ? r[hi][2 * vh + 1] : r[hi][2 * vh], 2);
            const int jj0 = 4 * J + 2 * h;
            *reinterpret_cast<double2*>(cellp + (k + (lo ? 0 : 1)) * NS + jj0) =
                lo ? make_double2(r[hi][2 * vh], other) : make_double2(other, r[hi][2 * vh + 1]);
          }
        }
      }
      fence_proxy_async();  // generic-proxy slab writes -> visible to the TMA unit
      mbar_arrive1(&slabFull[gi % NSLAB]);
      BZ_MARK(it, 6 + cdi, tid == 0);
      if (issuer) {
        // the slowest warp gates only this (lightly loaded) warp; the others
        // run up to two blocks ahead
        BZ_T0();
        mbar_wait(&slabFull[gi % NSLAB], (uint32_t)((gi / NSLAB) & 1));
        BZ_ACC(it, 15);
        slab_store(&amap, slab, d * NS, c * NS, (int)c0, acc);
        bulk_commit();
        if (gi >= 2) {
          bulk_wait_read2();  // block gi-2 has left its slab
          mbar_arrive1(&slabEmpty[(gi - 2) % NSLAB]);
        }
      }
    }
    if (issuer && it + 1 < my_tiles) {
      // slabs 0 and 1 (stores of steps 6, 7) read out -> first stages of the next tile
      BZ_MARK(it, 17, true);
      bulk_wait_read1();
      BZ_MARK(it, 18, true);
      for (int k = 0; k < RING_LA; ++k) {
        const long G = (it + 1) * KS2 + k;
        mbar_wait(&rEmpty[G % NRING], (uint32_t)(((G / NRING) - 1) & 1));
        ring_issue(G);
      }
    }
    if (it + 2 < my_tiles) nbar_arrive(BAR_EMPTY + b, THREADS);
  }
#endif
  if (issuer) bulk_wait0();
}

// ---------------------------------------------------------------------------
// host tables
// ---------------------------------------------------------------------------
bool burgers_supported(int nq, int ns) { return ns == bz::NS && nq > 0; }

int burgers_tables(int nq, const double* W, const double* B, const double* D, double* out) {
  // out = [S fragments | R2 fragments | Dn]
  using namespace bz;
  const int Q = nq;
  auto Bv = [&](int q, int j) { return B[(size_t)q * NS + j]; };
  auto Dv = [&](int a, int q, int j) { return D[((size_t)a * Q + q) * NS + j]; };
  // column (upper block ub, half h, col) -> (j, k): jj = 2h + col/4, kk = col%4
  auto jk_of = [&](int ub, int h, int col, int* j, int* k) {
    *j = 4 * bz_J(ub) + 2 * h + col / 4;
    *k = 4 * bz_K(ub) + col % 4;
  };
  // ---- orthonormal basis Psi of span{D_a[:, n]} (pivoted modified Gram-Schmidt)
  std::vector<std::vector<double>> res(3 * NS, std::vector<double>(Q));
  double maxn = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int n = 0; n < NS; ++n) {
      double s = 0.0;
      for (int q = 0; q < Q; ++q) {
        res[a * NS + n][q] = Dv(a, q, n);
        s += Dv(a, q, n) * Dv(a, q, n);
      }
      maxn = std::max(maxn, std::sqrt(s));
    }
  std::vector<std::vector<double>> psi;
  for (;;) {
    int p = -1;
    double best = 0.0;
    for (int i = 0; i < 3 * NS; ++i) {
      double s = 0.0;
      for (int q = 0; q < Q; ++q) s += res[i][q] * res[i][q];
      if (s > best) best = s, p = i;
    }
    if (p < 0 || std::sqrt(best) <= 1e-10 * maxn) break;
    if ((int)psi.size() == RMAX) return -1;
    std::vector<double> v = res[p];
    for (int pass = 0; pass < 2; ++pass)
      for (const auto& b : psi) {
        double dot = 0.0;
        for (int q = 0; q < Q; ++q) dot += b[q] * v[q];
        for (int q = 0; q < Q; ++q) v[q] -= dot * b[q];
      }
    double nv = 0.0;
    for (int q = 0; q < Q; ++q) nv += v[q] * v[q];
    nv = std::sqrt(nv);
    for (int q = 0; q < Q; ++q) v[q] /= nv;
    for (auto& r : res) {
      double dot = 0.0;
      for (int q = 0; q < Q; ++q) dot += v[q] * r[q];
      for (int q = 0; q < Q; ++q) r[q] -= dot * v[q];
    }
    psi.push_back(v);
  }
  const int rank = (int)psi.size();
  // Dn_a = Psi^T D_a; check D_a == Psi Dn_a
  double* Dn = out + S_DBL + R2_DBL;
  for (int i = 0; i < DN_DBL; ++i) Dn[i] = 0.0;
  double err = 0.0, amax = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int n = 0; n < NS; ++n) {
      for (int m = 0; m < rank; ++m) {
        double s = 0.0;
        for (int q = 0; q < Q; ++q) s += psi[m][q] * Dv(a, q, n);
        Dn[(a * DNR + m) * NS + n] = s;
      }
      for (int q = 0; q < Q; ++q) {
        double s = 0.0;
        for (int m = 0; m < rank; ++m) s += psi[m][q] * Dn[(a * DNR + m) * NS + n];
        err = std::max(err, std::fabs(s - Dv(a, q, n)));
        amax = std::max(amax, std::fabs(Dv(a, q, n)));
      }
    }
  if (err > 1e-12 * std::max(amax, 1.0)) return -1;
  // S fragments: b = S[m = 4ks + t][col g]
  for (int ub = 0; ub < NBU; ++ub)
    for (int ks = 0; ks < KS1; ++ks)
      for (int h = 0; h < 2; ++h)
        for (int lane = 0; lane < 32; ++lane) {
          const int g = lane >> 2, t = lane & 3, m = ks * 4 + t;
          int j, k;
          jk_of(ub, h, g, &j, &k);
          double s = 0.0;
          if (m < rank)
            for (int q = 0; q < Q; ++q) s += W[q] * psi[m][q] * Bv(q, j) * Bv(q, k);
          out[((ub * KS1 + ks) * 2 + h) * 32 + lane] = s;
        }
  // R2[alpha][j][k]
  std::vector<double> R2((size_t)KS2 * 4 * NS * NS, 0.0);
  for (int al = 0; al < 67; ++al)
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
          } else {
            v = Bv(q, j) * Bv(q, k);
          }
          s += W[q] * v;
        }
        R2[((size_t)al * NS + j) * NS + k] = s;
      }
  double* r2 = out + S_DBL;
  for (int ub = 0; ub < NBU; ++ub) {
    const bool off = bz_J(ub) != bz_K(ub);
    for (int ks = 0; ks < KS2; ++ks)
      for (int h = 0; h < 2; ++h)
        for (int lane = 0; lane < 32; ++lane) {
          const int g = lane >> 2, t = lane & 3, al = ks * 4 + t;
          int j, k;
          jk_of(ub, h, g, &j, &k);
          // direct tile: C[j][k]; mirror tile: the lane writing (k, j) needs C[k][j]
          // [ks][pair][32][2]: direct pair ub, mirror pair 15 + off index
          r2[((ks * NPAIR + ub) * 32 + lane) * 2 + h] = R2[((size_t)al * NS + j) * NS + k];
          if (off)
            r2[((ks * NPAIR + NBU + bz_off_index(ub)) * 32 + lane) * 2 + h] =
                R2[((size_t)al * NS + k) * NS + j];
        }
  }
  return rank;
}

size_t burgers_table_doubles() { return bz::S_DBL + bz::R2_DBL + bz::DN_DBL; }

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace

cudaError_t launch_burgers(int ns, long E, const double* coords, const double* coef,
                           const double* tab, double nu, double dt, double* A, int acc,
                           cudaStream_t s) {
  if (ns != bz::NS) return cudaErrorInvalidValue;
  if (E <= 0) return cudaSuccess;
  if (E > 0x7fffffffL) return cudaErrorInvalidValue;
  static const char once_key = 0;  // one per (kernel instantiation, device)
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(burgers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bz::SMEM);
    if (e != cudaSuccess) return e;
    return cudaSuccess;
  });
  if (e0 != cudaSuccess) return e0;
  auto encode = encode_fn();
  if (!encode) return cudaErrorNotSupported;
  // cuTensorMapEncodeTiled is a driver call: it needs the device's context current in
  // THIS host thread, which a thread whose first CUDA call is this launch does not have
  // yet (tests/test_gpu_robust.py::test_first_launch_race_fresh_process)
  int dev = 0;
  cudaError_t ec = cudaGetDevice(&dev);
  if (ec == cudaSuccess) ec = cudaSetDevice(dev);
  if (ec != cudaSuccess) return ec;
  // A_e as a 3D tensor [E][60 rows][60 cols]; box = one (c,d) block of 16 cells
  CUtensorMap map;
  const cuuint64_t dims[3] = {(cuuint64_t)bz::N, (cuuint64_t)bz::N, (cuuint64_t)E};
  const cuuint64_t strides[2] = {bz::N * sizeof(double), (cuuint64_t)bz::N * bz::N * sizeof(double)};
  const cuuint32_t box[3] = {bz::NS, bz::NS, bz::CELLS};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const long ntiles = (E + bz::CELLS - 1) / bz::CELLS;
  const long nsm = num_sms();
  const int grid = (int)(ntiles < nsm ? ntiles : nsm);
  burgers_kernel<<<grid, bz::THREADS, bz::SMEM, s>>>(map, E, coords, coef, tab, nu, dt, acc);
  return cudaGetLastError();
}

}  // namespace femgpu
