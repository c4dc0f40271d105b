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
//    operands -- g_j = K^T grad phi_j (elasticity), plus h_j = F g_j
//    (St Venant-Kirchhoff) -- computed once per chunk of
//    quadrature points, stored cell-fastest (lanes of one (j,k) tile read
//    consecutive addresses; j-stride padded so neighbouring tiles of a warp
//    hit alternate bank halves);
//  * every (c,d) component block of a (j,k) pair is a rank-2/3 update of these
//    records (component-blocked vector basis: the zero padding of the FFC
//    tables, zeroskip.cpp's concept, never enters the arithmetic):
//      elasticity  A(c,d) += mu' g_j[d] g_k[c] + lam' g_j[c] g_k[d] + d_cd mu' g_j.g_k
//      SVK         A(c,d) += lam' h_j[c] h_k[d] + mu' h_k[c] h_j[d]
//                            + mu' (F F^T)_cd g_j.g_k + d_cd s_j.g_k
//    where the stress term s_j.g_k = g_k^T (w'S) g_j needs no record of its own:
//    with S = lam tr(E) I + 2 mu E and 2E = F^T F - I it is
//      s_j.g_k = sig g_j.g_k + mu' h_j.h_k,   sig = w'(lam tr E - mu)
//    (sig joins the diagonal of the F F^T coefficients; mu' h_j.h_k is one more
//    dot product per pair of operands the accumulation loads anyway), so a record
//    holds g | h (6 doubles) instead of g | h | s (9): 16 % fewer shared-memory
//    operand loads per (j,k) tile and point, 30 % fewer record stores;
//  * A_e is symmetric for both forms: only j<=k pairs are accumulated (2x2
//    register tiles over the upper triangle of the 10x10 (j,k) grid), one
//    (cell, tile) per accumulating thread, independent FMA passes;
//  * element matrices are staged in shared memory (cell stride 902 doubles:
//    conflict-free 16-byte stores) and written by TMA bulk copies
//    (cp.async.bulk, or cp.reduce.async.bulk .add.f64 for the += contract).
//
// CTA organisations (chosen per form by measurement, profiles/):
//  * pair_ws_kernel  (elasticity): warp-specialised -- 2 producer warps build
//    the records of the next tile into a double buffer (mbarrier full/empty)
//    while 4 consumer warps accumulate; 2 CTAs per SM;
//  * pair_svk_ws_kernel (SVK): warp-specialised with a deeper ring -- 3 producer
//    warps run the heavier per-point setup (F, tr E, F F^T, h_j, G_jk per (cell, q))
//    into a 4-slot ring of 2-point stages while 8 consumer warps (off-diagonal and
//    diagonal tiles in warps of their own) accumulate; one CTA of 16 cells per SM
//    pools the shared memory for the ring (c4: 1.107 ms);
//  * pair_flat_kernel (SVK before, PAIR_SVK_WS=0): every thread takes part in each
//    phase; 2 CTAs per SM overlap one CTA's setup with the other's FMA stream
//    (c4 1.31 ms against 1.25 ms for the round-1 ring kernel).
//
// SVK accumulates each 3x3 (c,d) block as its symmetric and antisymmetric parts
// (pair_point, svk_unfold): 27 instead of 33 FP64 instructions per pair and point.
#include <cstring>

#include "common.cuh"
#include "femgpu_internal.h"
#include "../../include/femgpu.h"

#ifndef PAIR_QUNROLL
#define PAIR_QUNROLL 4  // q-loop unroll of the accumulate phase (measured: 1.56 -> 1.48 ms on c4)
#endif
#ifndef PAIR_WS_QUNROLL
#define PAIR_WS_QUNROLL 8  // elasticity consumers (Q = 8; measured 1.081 -> 1.011 ms on c3 vs 1)
#endif
#ifndef PAIR_FLAT_WARP_CELLS
#define PAIR_FLAT_WARP_CELLS 0  // warp-owned cells in the flat (SVK) kernel: 1.48 vs 1.42 ms on c4
#endif
#ifndef PAIR_ELAS_FLAT
#define PAIR_ELAS_FLAT 0
#endif
#ifndef PAIR_FLAT_CTAS
#define PAIR_FLAT_CTAS 2  // CTAs per SM of the flat (SVK) kernel
#endif
#ifndef PAIR_SVK_QC
#define PAIR_SVK_QC 14  // SVK quadrature points per chunk (14 -> 112 of 128 threads busy in the setup)
#endif
#ifndef PAIR_SVK_WS
#define PAIR_SVK_WS 1  // SVK: warp-specialised kernel (1) or the flat one (0)
#endif
#ifndef PAIR_SVK_CELLS
#define PAIR_SVK_CELLS 16  // SVK ws: cells per CTA tile (8: 2 CTAs per SM, 16: one)
#endif
#ifndef PAIR_SVK_SLOTS
#define PAIR_SVK_SLOTS (PAIR_SVK_GREC ? 4 : 5)  // SVK ws: record ring slots (0: one per producer warp)
#endif
#ifndef PAIR_SVK_PW
#define PAIR_SVK_PW 3  // SVK ws: producer warps that build ring stages (of 4)
#endif
#ifndef PAIR_SVK_QUNROLL
#define PAIR_SVK_QUNROLL 2  // SVK ws consumers: unroll of a stage's points (1: 1.147 vs 1.107 ms)
#endif
#ifndef PAIR_SVK_GREC
#define PAIR_SVK_GREC 1  // SVK ws: records h_j + G_jk (producers do the g_j.g_k) instead of g_j | h_j
#endif
#ifndef PAIR_SVK_PARAMTAB
#define PAIR_SVK_PARAMTAB PAIR_SVK_GREC  // SVK ws: W | D | P as a kernel parameter (constant bank)
                                         // instead of smem (frees 7.6 KB for the G records)
#endif
#ifndef PAIR_ABL  // development ablations of pair_ws_kernel: bit 0 no accumulate, bit 1 no store,
                  // bit 2 no records, bit 3 no geometry, bit 4 no staging
                  // (pair_flat_kernel: bit 0 no accumulate, bit 2 no per-point setup)
#define PAIR_ABL 0
#endif

namespace femgpu {

constexpr int kPairQUnroll = PAIR_QUNROLL;
constexpr int kPairWsQUnroll = PAIR_WS_QUNROLL;
constexpr int kSvkQUnroll = PAIR_SVK_QUNROLL;

template <int KIND, int NS, int Q>
struct PairShape {
  static constexpr bool SVK = (KIND == FEMGPU_HYPERELASTICITY);
  static constexpr int N = 3 * NS;                       // element matrix N x N
  static constexpr int NJ = NS / 2;                      // 2-wide j/k groups
  static constexpr int NTILE = NJ * (NJ + 1) / 2;        // 2x2 tiles on/above the diagonal
  static constexpr int CELLS = 8;                        // cells per CTA tile
  static constexpr int ACC = 128;                        // accumulating threads: 8 x 16 slots
  static constexpr bool FLAT = SVK || PAIR_ELAS_FLAT;    // organisation (see header)
  static constexpr int PROD = FLAT ? 0 : 64;             // producer threads (ws kernel only)
  static constexpr int THREADS = ACC + PROD;
  static constexpr int CTAS_PER_SM = FLAT ? PAIR_FLAT_CTAS : 2;
  static constexpr int NCOEF = SVK ? 3 * NS + 8 : 8;
  static constexpr int QC = SVK ? PAIR_SVK_QC : Q;       // quadrature points per chunk
  static constexpr int NCHUNK = (Q + QC - 1) / QC;
  static constexpr int RECD = SVK ? 6 : 3;               // per (q,j): g | h (SVK), g
  static constexpr int QSD = SVK ? 8 : 2;                // per q: al, be | F F^T + sig (6)
  // ws (elasticity): each warp owns WCELLS cells of the tile (see pair_slot)
  static constexpr bool WARP_CELLS = !FLAT || PAIR_FLAT_WARP_CELLS;
  static constexpr int WCELLS = CELLS / (ACC / 32);
  // j-stride of a record buffer.  flat: RECD*CELLS + 4 doubles, so the k-side loads
  // of the (j,k) tiles sharing a warp (k0 two apart) fall in alternate bank halves;
  // ws: == 1 mod 8, so the 5 even k0 rows x WCELLS cells of a warp's load hit
  // distinct banks (one wavefront)
  static constexpr int JS = WARP_CELLS ? RECD * CELLS + 1 : RECD * CELLS + 4;
  static constexpr int REC_DBL = QC * (NS * JS + QSD * CELLS);  // one record buffer
  static constexpr int CSTRIDE = N * N + 2;              // staging stride: (stride/2) odd
  static constexpr int STG_DBL = CELLS * CSTRIDE;
  static constexpr int TAB0 = Q + 3 * Q * NS + 4 * Q;    // W | D | P
  static constexpr int TAB = (TAB0 + 1) / 2 * 2;
  static constexpr int CELLD = 10;                       // K(9), adet
  // ws: coefficient rows padded to an odd stride (the producer's per-(cell, q) reads
  // of 8 cells' rows are conflict-free)
  static constexpr int CF = !FLAT ? NCOEF + 1 : NCOEF;
  static constexpr int IN_DBL = CELLS * (12 + CF);       // raw inputs
  static constexpr int HEAD = TAB + CELLS * CELLD + (FLAT ? 1 : 2) * IN_DBL;  // ws: double-buffered inputs
  // ws: two record buffers + separate staging; flat: one record buffer aliasing staging
  static constexpr int BODY = FLAT ? (REC_DBL > STG_DBL ? REC_DBL : STG_DBL)
                                   : 2 * REC_DBL + STG_DBL;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)HEAD + BODY) + 4 * sizeof(uint64_t);
  static_assert(NS % 2 == 0, "2x2 tiling needs an even number of scalar dofs");
  static_assert(CELLS * (NTILE + 1) <= ACC, "one (cell, tile) per accumulating thread");
  static_assert(!WARP_CELLS || (WCELLS * (ACC / 32) == CELLS && WCELLS * NTILE <= 32),
                "ws: warp-owned cells");
  static_assert((CSTRIDE / 2) % 2 == 1, "conflict-free staging stride");
  static_assert(HEAD % 2 == 0 && REC_DBL % 2 == 0, "16-byte aligned buffers");
};

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// (cell, tile) of an accumulating thread: tile t -> upper 2x2 block (TJ, TK)
struct PairSlot {
  int cell, j0, k0;
  bool active, diag;
};
// ws lane -> (cell of the warp) * 16 + tile for NS = 10, 2 cells per warp and a
// staging cell stride of 902 doubles: the 16-byte staging stores of every quarter-warp
// hit distinct bank groups, and of the whole warp at most ceil(bytes / 128) per group
// (direct and mirrored; searched offline; -1 idle)
__constant__ signed char c_ws_lane10[32] = {7,  6,  17, 9,  18, 2,  16, 30, 14, 5,  24,
                                            13, 22, 1,  8,  11, 29, 4,  20, 28, 26, 12,
                                            19, 3,  10, 27, 25, 23, 21, 0,  -1, -1};

// flat kernel: cell = tid % CELLS (a warp spans all cells of the tile);
// ws kernel: warp w owns cells WCELLS*w .. WCELLS*w + WCELLS-1 (one lane per (cell, tile)),
// so a warp stages and stores its cells without waiting for the other warps
template <class Sh>
__device__ __forceinline__ PairSlot pair_slot(int tid) {
  PairSlot s;
  int my_tile;
  if constexpr (Sh::WARP_CELLS && Sh::NJ == 5 && Sh::WCELLS == 2 && Sh::CSTRIDE % 16 == 6) {
    const int code = c_ws_lane10[tid & 31];
    s.cell = (tid >> 5) * Sh::WCELLS + (code >= 0 ? code >> 4 : 0);
    my_tile = code & 15;
    s.active = code >= 0;
  } else if constexpr (Sh::WARP_CELLS) {
    const int lane = tid & 31;
    s.cell = (tid >> 5) * Sh::WCELLS + lane / Sh::NTILE;
    my_tile = lane % Sh::NTILE;
    s.active = lane < Sh::WCELLS * Sh::NTILE;
  } else {
    s.cell = tid % Sh::CELLS;
    my_tile = tid / Sh::CELLS;
    s.active = my_tile < Sh::NTILE;
  }
  int TJ = 0, TK = 0, t = s.active ? my_tile : 0;
  for (int J = 0; J < Sh::NJ; ++J) {
    const int len = Sh::NJ - J;
    if (t < len) {
      TJ = J;
      TK = J + t;
      break;
    }
    t -= len;
  }
  s.j0 = 2 * TJ;
  s.k0 = 2 * TK;
  s.diag = TJ == TK;
  return s;
}

// Accumulate one quadrature point's records into the thread's 2x2 tile.
template <class Sh>
__device__ __forceinline__ void pair_point(double (&a4)[2][2][3][3], double (&t1)[2][2],
                                           const double* rq, const double* qs, int j0, int k0) {
  constexpr int CELLS = Sh::CELLS, JS = Sh::JS;
  const double lq = qs[0], mq = qs[CELLS];
  double gk[2][3];
#pragma unroll
  for (int y = 0; y < 2; ++y)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) gk[y][bb] = rq[(k0 + y) * JS + bb * CELLS];
  if constexpr (!Sh::SVK) {
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      double u[3], v[3];
#pragma unroll
      for (int bb = 0; bb < 3; ++bb) {
        const double gj = rq[(j0 + x) * JS + bb * CELLS];
        u[bb] = mq * gj;
        v[bb] = lq * gj;
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
      // mu' g_j.g_k accumulates over q on its own; added to the (c,c) entries once
#pragma unroll
      for (int y = 0; y < 2; ++y)
        t1[x][y] = fma(u[0], gk[y][0], fma(u[1], gk[y][1], fma(u[2], gk[y][2], t1[x][y])));
    }
  } else {
    double hk[2][3];
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int bb = 0; bb < 3; ++bb) hk[y][bb] = rq[(k0 + y) * JS + (3 + bb) * CELLS];
    // Symmetric / antisymmetric split of each 3x3 (c,d) block (svk_unfold):
    //   lam h_j[c] h_k[d] + mu h_k[c] h_j[d] = al (h_j[c] h_k[d] + h_j[d] h_k[c])
    //                                        + be (h_j[c] h_k[d] - h_j[d] h_k[c]),
    // al = (lam'+mu')/2, be = (lam'-mu')/2; the mu' F F^T (g_j.g_k) term is symmetric.
    // a4[c][d] (c<=d) holds the symmetric part (diagonal halved), a4[d][c] (c<d) the
    // antisymmetric one: 27 instead of 33 FP64 instructions per (j,k) pair and point.
    // qs holds al, be, then mu' F F^T with its diagonal halved (setup), the diagonal
    // carrying sig/2 as well: the sig g_j.g_k part of the stress term s_j.g_k.  Its
    // other part, mu' h_j.h_k with mu' h_j = al h_j - be h_j, accumulates in t1.
    const double f00 = qs[2 * CELLS], f01 = qs[3 * CELLS], f02 = qs[4 * CELLS];
    const double f11 = qs[5 * CELLS], f12 = qs[6 * CELLS], f22 = qs[7 * CELLS];
    const double ff[3][3] = {{f00, f01, f02}, {f01, f11, f12}, {f02, f12, f22}};
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      double gj[3], ah[3], bh[3], mh[3];
      const double* r = rq + (j0 + ((PAIR_ABL & 32) ? 0 : x)) * JS;  // 32: timing ablation
#pragma unroll
      for (int bb = 0; bb < 3; ++bb) {
        gj[bb] = r[bb * CELLS];                // g_j
        const double h = r[(3 + bb) * CELLS];
        ah[bb] = lq * h;                       // al h_j
        bh[bb] = mq * h;                       // be h_j
        mh[bb] = ah[bb] - bh[bb];              // mu' h_j
      }
      double t2[2];
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        // mu' h_j.h_k accumulates over q on its own; added to the (c,c) entries once
        t1[x][y] = fma(mh[0], hk[y][0], fma(mh[1], hk[y][1], fma(mh[2], hk[y][2], t1[x][y])));
        t2[y] = gj[0] * gk[y][0] + gj[1] * gk[y][1] + gj[2] * gk[y][2];
      }
      // first terms: symmetric diagonal and off-diagonal, antisymmetric
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = c; d < 3; ++d) {
            a4[x][y][c][d] = fma(ah[c], hk[y][d], a4[x][y][c][d]);
            if (d > c) a4[x][y][d][c] = fma(bh[c], hk[y][d], a4[x][y][d][c]);
          }
      // second terms of the off-diagonal entries; F F^T term of the diagonal
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = c; d < 3; ++d) {
            if (d > c) {
              a4[x][y][c][d] = fma(ah[d], hk[y][c], a4[x][y][c][d]);
              a4[x][y][d][c] = fma(-bh[d], hk[y][c], a4[x][y][d][c]);
            } else {
              a4[x][y][c][c] = fma(t2[y], ff[c][c], a4[x][y][c][c]);
            }
          }
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = c + 1; d < 3; ++d) a4[x][y][c][d] = fma(t2[y], ff[c][d], a4[x][y][c][d]);
    }
  }
}

// SVK, one diagonal 2x2 tile (j0 = k0) of the ring kernel: the k side is the j side,
// so a point needs 12 record loads (g, h of j0, j0+1) and the 8 point scalars instead
// of 32, and only the pairs (j0,j0), (j0,j0+1), (j0+1,j0+1) are accumulated (87 FP64
// instructions against 126).  A self pair (j,j) has no antisymmetric part; a4[1][0]
// and t1[1][0] stay unused (pair_stage writes the (j0+1, j0) block as the mirror).
template <class Sh>
__device__ __forceinline__ void pair_point_diag(double (&a4)[2][2][3][3], double (&t1)[2][2],
                                                const double* rq, const double* qs, int j0) {
  constexpr int CELLS = Sh::CELLS, JS = Sh::JS;
  const double lq = qs[0], mq = qs[CELLS];
  const double f00 = qs[2 * CELLS], f01 = qs[3 * CELLS], f02 = qs[4 * CELLS];
  const double f11 = qs[5 * CELLS], f12 = qs[6 * CELLS], f22 = qs[7 * CELLS];
  const double ff[3][3] = {{f00, f01, f02}, {f01, f11, f12}, {f02, f12, f22}};
  double g[2][3], h[2][3], ah[2][3], bh[2][3], mh[2][3];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      g[x][bb] = rq[(j0 + x) * JS + bb * CELLS];
      h[x][bb] = rq[(j0 + x) * JS + (3 + bb) * CELLS];
    }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      ah[x][bb] = lq * h[x][bb];
      bh[x][bb] = mq * h[x][bb];
      mh[x][bb] = ah[x][bb] - bh[x][bb];
    }
  // self pairs (x, x)
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    t1[x][x] = fma(mh[x][0], h[x][0], fma(mh[x][1], h[x][1], fma(mh[x][2], h[x][2], t1[x][x])));
    const double t2 = g[x][0] * g[x][0] + g[x][1] * g[x][1] + g[x][2] * g[x][2];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = c; d < 3; ++d) {
        a4[x][x][c][d] = fma(ah[x][c], h[x][d], a4[x][x][c][d]);
        if (d > c) a4[x][x][c][d] = fma(ah[x][d], h[x][c], a4[x][x][c][d]);
        a4[x][x][c][d] = fma(t2, ff[c][d], a4[x][x][c][d]);
      }
  }
  // the mixed pair (j0, j0+1): as pair_point
  {
    t1[0][1] = fma(mh[0][0], h[1][0], fma(mh[0][1], h[1][1], fma(mh[0][2], h[1][2], t1[0][1])));
    const double t2 = g[0][0] * g[1][0] + g[0][1] * g[1][1] + g[0][2] * g[1][2];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = c; d < 3; ++d) {
        a4[0][1][c][d] = fma(ah[0][c], h[1][d], a4[0][1][c][d]);
        if (d > c) a4[0][1][d][c] = fma(bh[0][c], h[1][d], a4[0][1][d][c]);
      }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = c; d < 3; ++d) {
        if (d > c) {
          a4[0][1][c][d] = fma(ah[0][d], h[1][c], a4[0][1][c][d]);
          a4[0][1][d][c] = fma(-bh[0][d], h[1][c], a4[0][1][d][c]);
        }
        a4[0][1][c][d] = fma(t2, ff[c][d], a4[0][1][c][d]);
      }
  }
}

// SVK ring kernel with G records (PAIR_SVK_GREC): the producers store, per (cell,
// point), h_j (3 per j) and the 55 G_jk = g_j.g_k instead of g_j | h_j, so a 2x2
// tile's point reads h of its two j and two k rows, its 4 G values and the 8 point
// scalars (24 loads instead of 32) and skips the 12 FP64 instructions of its four
// g_j.g_k; the dot products move to the producer warps, which wait on the ring
// otherwise.  rq: this cell's h records (j stride JS, component stride CELLS),
// gq: its G of pairs p (stride CELLS), qs: its point scalars.
template <class Sh>
__device__ __forceinline__ void svk_point_g(double (&a4)[2][2][3][3], double (&t1)[2][2],
                                            const double* rq, const double* gq,
                                            const double* qs, int j0, int k0,
                                            const int (&p)[2][2]) {
  constexpr int CELLS = Sh::CELLS, JS = Sh::JS;
  const double lq = qs[0], mq = qs[CELLS];
  const double f00 = qs[2 * CELLS], f01 = qs[3 * CELLS], f02 = qs[4 * CELLS];
  const double f11 = qs[5 * CELLS], f12 = qs[6 * CELLS], f22 = qs[7 * CELLS];
  const double ff[3][3] = {{f00, f01, f02}, {f01, f11, f12}, {f02, f12, f22}};
  double hk[2][3];
#pragma unroll
  for (int y = 0; y < 2; ++y)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) hk[y][bb] = rq[(k0 + y) * JS + bb * CELLS];
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    double ah[3], bh[3], mh[3];
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      const double h = rq[(j0 + x) * JS + bb * CELLS];
      ah[bb] = lq * h;
      bh[bb] = mq * h;
      mh[bb] = ah[bb] - bh[bb];
    }
    double t2[2];
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      t1[x][y] = fma(mh[0], hk[y][0], fma(mh[1], hk[y][1], fma(mh[2], hk[y][2], t1[x][y])));
      t2[y] = gq[p[x][y] * CELLS];
    }
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = c; d < 3; ++d) {
          a4[x][y][c][d] = fma(ah[c], hk[y][d], a4[x][y][c][d]);
          if (d > c) a4[x][y][d][c] = fma(bh[c], hk[y][d], a4[x][y][d][c]);
        }
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = c; d < 3; ++d) {
          if (d > c) {
            a4[x][y][c][d] = fma(ah[d], hk[y][c], a4[x][y][c][d]);
            a4[x][y][d][c] = fma(-bh[d], hk[y][c], a4[x][y][d][c]);
          }
          a4[x][y][c][d] = fma(t2[y], ff[c][d], a4[x][y][c][d]);
        }
  }
}

// The diagonal tile of svk_point_g (pair_point_diag with G records): 17 loads.
template <class Sh>
__device__ __forceinline__ void svk_point_g_diag(double (&a4)[2][2][3][3], double (&t1)[2][2],
                                                 const double* rq, const double* gq,
                                                 const double* qs, int j0, const int (&p)[2][2]) {
  constexpr int CELLS = Sh::CELLS, JS = Sh::JS;
  const double lq = qs[0], mq = qs[CELLS];
  const double f00 = qs[2 * CELLS], f01 = qs[3 * CELLS], f02 = qs[4 * CELLS];
  const double f11 = qs[5 * CELLS], f12 = qs[6 * CELLS], f22 = qs[7 * CELLS];
  const double ff[3][3] = {{f00, f01, f02}, {f01, f11, f12}, {f02, f12, f22}};
  double h[2][3], ah[2][3], bh[2][3], mh[2][3];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      h[x][bb] = rq[(j0 + x) * JS + bb * CELLS];
      ah[x][bb] = lq * h[x][bb];
      bh[x][bb] = mq * h[x][bb];
      mh[x][bb] = ah[x][bb] - bh[x][bb];
    }
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    t1[x][x] = fma(mh[x][0], h[x][0], fma(mh[x][1], h[x][1], fma(mh[x][2], h[x][2], t1[x][x])));
    const double t2 = gq[p[x][x] * CELLS];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = c; d < 3; ++d) {
        a4[x][x][c][d] = fma(ah[x][c], h[x][d], a4[x][x][c][d]);
        if (d > c) a4[x][x][c][d] = fma(ah[x][d], h[x][c], a4[x][x][c][d]);
        a4[x][x][c][d] = fma(t2, ff[c][d], a4[x][x][c][d]);
      }
  }
  {
    t1[0][1] = fma(mh[0][0], h[1][0], fma(mh[0][1], h[1][1], fma(mh[0][2], h[1][2], t1[0][1])));
    const double t2 = gq[p[0][1] * CELLS];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = c; d < 3; ++d) {
        a4[0][1][c][d] = fma(ah[0][c], h[1][d], a4[0][1][c][d]);
        if (d > c) a4[0][1][d][c] = fma(bh[0][c], h[1][d], a4[0][1][d][c]);
      }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = c; d < 3; ++d) {
        if (d > c) {
          a4[0][1][c][d] = fma(ah[0][d], h[1][c], a4[0][1][c][d]);
          a4[0][1][d][c] = fma(-bh[0][d], h[1][c], a4[0][1][d][c]);
        }
        a4[0][1][c][d] = fma(t2, ff[c][d], a4[0][1][c][d]);
      }
  }
}

// SVK: symmetric (upper, diagonal halved) / antisymmetric (lower) parts -> the block.
__device__ __forceinline__ void svk_unfold(double (&a4)[2][2][3][3]) {
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a4[x][y][c][c] *= 2.0;
#pragma unroll
        for (int d = c + 1; d < 3; ++d) {
          const double s = a4[x][y][c][d], n = a4[x][y][d][c];
          a4[x][y][c][d] = s + n;
          a4[x][y][d][c] = s - n;
        }
      }
    }
}

// Per (cell, quadrature point) setup, one thread: lam', mu' (and, SVK: F = I + grad w,
// tr E, mu' F F^T, sig), then the records of the NS basis functions at q: g_j = K^T D phi_j
// (elasticity), plus h_j = F g_j (SVK).  qs / rec: this cell's
// per-point scalars (stride CELLS) and records (j stride JS, component stride CELLS).
template <bool SVK, int NS, int Q, int CELLS, int JS, int NCOEF, class TW, class TD, class TP>
__device__ __forceinline__ void pair_point_setup(const double* K, const double* cf, bool valid,
                                                 int q, const TW& sW, const TD& sD, const TP& sP,
                                                 double* qs, double* rec) {
  auto cv = [&](int r) -> double { return valid ? cf[r] : 0.0; };
  constexpr int CO = SVK ? 3 * NS : 0;  // offset of mu, lam in the dofs
  double muq = 0, lamq = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    muq += cv(CO + m) * sP[q * 4 + m];
    lamq += cv(CO + 4 + m) * sP[q * 4 + m];
  }
  const double wq = sW[q] * K[9];
  double Kr[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Kr[i] = K[i];
  if constexpr (!SVK) {
    qs[0 * CELLS] = lamq * wq;
    qs[1 * CELLS] = muq * wq;
#pragma unroll 2
    for (int j = 0; j < NS; ++j) {
      double* rr = rec + j * JS;
#pragma unroll
      for (int b = 0; b < 3; ++b)
        rr[b * CELLS] = Kr[0 * 3 + b] * sD[(0 * Q + q) * NS + j] +
                        Kr[1 * 3 + b] * sD[(1 * Q + q) * NS + j] +
                        Kr[2 * 3 + b] * sD[(2 * Q + q) * NS + j];
    }
  } else {
    // al, be of the symmetric / antisymmetric split (pair_point, svk_unfold)
    qs[0 * CELLS] = 0.5 * (lamq + muq) * wq;
    qs[1 * CELLS] = 0.5 * (lamq - muq) * wq;
    // reference derivatives of the NS basis functions at q, read once for grad w
    // and the records
    double dq[3][NS];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int m = 0; m < NS; ++m) dq[a][m] = sD[(a * Q + q) * NS + m];
    double F[3][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
      double gr[3] = {0, 0, 0};  // reference gradient of w_cc
#pragma unroll
      for (int m = 0; m < NS; ++m) {
        const double wm = cv(cc * NS + m);
#pragma unroll
        for (int a = 0; a < 3; ++a) gr[a] += wm * dq[a][m];
      }
#pragma unroll
      for (int b = 0; b < 3; ++b)
        F[cc][b] = (cc == b ? 1.0 : 0.0) + gr[0] * Kr[0 * 3 + b] + gr[1] * Kr[1 * 3 + b] +
                   gr[2] * Kr[2 * 3 + b];
    }
    // tr E, E = (F^T F - I)/2; the stress term s_j.g_k = g_k^T w'S g_j with
    // S = lam tr(E) I + 2 mu E = (lam tr E - mu) I + mu F^T F becomes
    // sig g_j.g_k + mu' h_j.h_k, sig = w'(lam tr E - mu), mu' = w' mu (pair_point)
    double trE = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
      trE += 0.5 * ((F[0][a] * F[0][a] + F[1][a] * F[1][a] + F[2][a] * F[2][a]) - 1.0);
    // mu' F F^T (0,0),(0,1),(0,2),(1,1),(1,2),(2,2), pre-scaled for the accumulate
    // phase; diagonal halved (svk_unfold) and carrying sig/2
    const double mw = muq * wq, mh = 0.5 * mw, sh = 0.5 * (wq * (lamq * trE - muq));
    qs[2 * CELLS] = mh * (F[0][0] * F[0][0] + F[0][1] * F[0][1] + F[0][2] * F[0][2]) + sh;
    qs[3 * CELLS] = mw * (F[0][0] * F[1][0] + F[0][1] * F[1][1] + F[0][2] * F[1][2]);
    qs[4 * CELLS] = mw * (F[0][0] * F[2][0] + F[0][1] * F[2][1] + F[0][2] * F[2][2]);
    qs[5 * CELLS] = mh * (F[1][0] * F[1][0] + F[1][1] * F[1][1] + F[1][2] * F[1][2]) + sh;
    qs[6 * CELLS] = mw * (F[1][0] * F[2][0] + F[1][1] * F[2][1] + F[1][2] * F[2][2]);
    qs[7 * CELLS] = mh * (F[2][0] * F[2][0] + F[2][1] * F[2][1] + F[2][2] * F[2][2]) + sh;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      double g[3];
#pragma unroll
      for (int b = 0; b < 3; ++b)
        g[b] = Kr[0 * 3 + b] * dq[0][j] + Kr[1 * 3 + b] * dq[1][j] + Kr[2 * 3 + b] * dq[2][j];
      double* rr = rec + j * JS;
#pragma unroll
      for (int b = 0; b < 3; ++b) rr[b * CELLS] = g[b];
#pragma unroll
      for (int a = 0; a < 3; ++a) rr[(3 + a) * CELLS] = F[a][0] * g[0] + F[a][1] * g[1] + F[a][2] * g[2];
    }
  }
}

// Per (cell, point) setup of the SVK ring kernel with G records: the point scalars as
// pair_point_setup, then h_j = F g_j (records, j stride JS) and G_jk = g_j.g_k for the
// j <= k pairs (gq, pair stride CELLS).  TW/TD/TP: W | D | P tables.
template <int NS, int Q, int CELLS, int JS, class TW, class TD, class TP>
__device__ __forceinline__ void svk_setup_g(const double* K, const double* cf, bool valid, int q,
                                            const TW& sW, const TD& sD, const TP& sP, double* qs,
                                            double* rec, double* gq) {
  auto cv = [&](int r) -> double { return valid ? cf[r] : 0.0; };
  constexpr int CO = 3 * NS;
  double muq = 0, lamq = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    muq += cv(CO + m) * sP[q * 4 + m];
    lamq += cv(CO + 4 + m) * sP[q * 4 + m];
  }
  const double wq = sW[q] * K[9];
  double Kr[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Kr[i] = K[i];
  qs[0 * CELLS] = 0.5 * (lamq + muq) * wq;
  qs[1 * CELLS] = 0.5 * (lamq - muq) * wq;
  double dq[3][NS];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int m = 0; m < NS; ++m) dq[a][m] = sD[(a * Q + q) * NS + m];
  double F[3][3];
#pragma unroll
  for (int cc = 0; cc < 3; ++cc) {
    double gr[3] = {0, 0, 0};
#pragma unroll
    for (int m = 0; m < NS; ++m) {
      const double wm = cv(cc * NS + m);
#pragma unroll
      for (int a = 0; a < 3; ++a) gr[a] += wm * dq[a][m];
    }
#pragma unroll
    for (int b = 0; b < 3; ++b)
      F[cc][b] = (cc == b ? 1.0 : 0.0) + gr[0] * Kr[0 * 3 + b] + gr[1] * Kr[1 * 3 + b] +
                 gr[2] * Kr[2 * 3 + b];
  }
  double trE = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    trE += 0.5 * ((F[0][a] * F[0][a] + F[1][a] * F[1][a] + F[2][a] * F[2][a]) - 1.0);
  const double mw = muq * wq, mh = 0.5 * mw, sh = 0.5 * (wq * (lamq * trE - muq));
  qs[2 * CELLS] = mh * (F[0][0] * F[0][0] + F[0][1] * F[0][1] + F[0][2] * F[0][2]) + sh;
  qs[3 * CELLS] = mw * (F[0][0] * F[1][0] + F[0][1] * F[1][1] + F[0][2] * F[1][2]);
  qs[4 * CELLS] = mw * (F[0][0] * F[2][0] + F[0][1] * F[2][1] + F[0][2] * F[2][2]);
  qs[5 * CELLS] = mh * (F[1][0] * F[1][0] + F[1][1] * F[1][1] + F[1][2] * F[1][2]) + sh;
  qs[6 * CELLS] = mw * (F[1][0] * F[2][0] + F[1][1] * F[2][1] + F[1][2] * F[2][2]);
  qs[7 * CELLS] = mh * (F[2][0] * F[2][0] + F[2][1] * F[2][1] + F[2][2] * F[2][2]) + sh;
  double g[NS][3];
#pragma unroll
  for (int j = 0; j < NS; ++j) {
#pragma unroll
    for (int b = 0; b < 3; ++b)
      g[j][b] = Kr[0 * 3 + b] * dq[0][j] + Kr[1 * 3 + b] * dq[1][j] + Kr[2 * 3 + b] * dq[2][j];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      rec[j * JS + a * CELLS] = F[a][0] * g[j][0] + F[a][1] * g[j][1] + F[a][2] * g[j][2];
  }
  int p = 0;
#pragma unroll
  for (int j = 0; j < NS; ++j)
#pragma unroll
    for (int k = j; k < NS; ++k, ++p)
      gq[p * CELLS] = g[j][0] * g[k][0] + g[j][1] * g[k][1] + g[j][2] * g[k][2];
}

// The q-summed scalar term (SVK mu' h_j.h_k, elasticity mu' g_j.g_k) enters the
// (c,c) entries of each (j,k) pair once.
__device__ __forceinline__ void add_t1(double (&a4)[2][2][3][3], const double (&t1)[2][2]) {
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int c = 0; c < 3; ++c) a4[x][y][c][c] += t1[x][y];
}

// The tile's symmetric half, mirrored, into the cell's staging row.
template <class Sh>
__device__ __forceinline__ void pair_stage(double* stg, const double (&a4)[2][2][3][3],
                                           const PairSlot& sl) {
  constexpr int N = Sh::N, NS = N / 3;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d)
        // row (c, j0+x), columns (d, k0..k0+1): one 16-byte store.  Diagonal tile:
        // entry (j0+1, k0) is the mirror of (j0, k0+1) (the lower triangle is the
        // mirrored upper one) -- folded into this store (ws), or stored apart (flat:
        // measured faster there)
        *reinterpret_cast<double2*>(&stg[(c * NS + sl.j0 + x) * N + d * NS + sl.k0]) =
            make_double2(Sh::WARP_CELLS && x == 1 && sl.diag ? a4[0][1][d][c] : a4[x][0][c][d],
                         a4[x][1][c][d]);
  if (!sl.diag) {
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d)
          // mirror: row (d, k0+y), columns (c, j0..j0+1)
          *reinterpret_cast<double2*>(&stg[(d * NS + sl.k0 + y) * N + c * NS + sl.j0]) =
              make_double2(a4[0][y][c][d], a4[1][y][c][d]);
  } else if constexpr (!Sh::WARP_CELLS) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) stg[(d * NS + sl.k0 + 1) * N + c * NS + sl.j0] = a4[0][1][c][d];
  }
}

// Staged element matrices -> global by the TMA engine (one thread issues).
template <class Sh>
__device__ __forceinline__ void pair_bulk_store(double* A, long c0, int nt, const double* stg,
                                                int acc) {
  constexpr int N = Sh::N;
  for (int c = 0; c < nt; ++c) {
    double* dst = A + (c0 + c) * (size_t)N * N;
    if (acc)
      bulk_s2g_add(dst, stg + c * Sh::CSTRIDE, N * N * 8);
    else
      bulk_s2g(dst, stg + c * Sh::CSTRIDE, N * N * 8);
  }
  bulk_commit();
}

__device__ __forceinline__ void zero_tile(double (&a4)[2][2][3][3]) {
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) a4[x][y][c][d] = 0.0;
}

// ============================================================================
// Elasticity: warp-specialised (2 producer warps, 4 consumer warps)
// ============================================================================
template <int NS, int Q>
__global__ void __launch_bounds__(PairShape<FEMGPU_ELASTICITY, NS, Q>::THREADS, 2)
    pair_ws_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                   const double* __restrict__ tab, double* __restrict__ A, int acc) {
  using Sh = PairShape<FEMGPU_ELASTICITY, NS, Q>;
  constexpr int CELLS = Sh::CELLS;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;
  double* sD = sW + Q;                      // [3][Q][NS]
  double* sP = sD + 3 * Q * NS;             // [Q][4]
  double* sCell = smem + Sh::TAB;           // [CELLS][CELLD]    (producer)
  double* sIn = sCell + CELLS * Sh::CELLD;  // [2][CELLS][12 | NCOEF]  (producer)
  double* sRec = sIn + 2 * Sh::IN_DBL;      // [2][REC_DBL]  producer -> consumers
  double* sStg = sRec + 2 * Sh::REC_DBL;    // [CELLS][CSTRIDE]  consumers -> TMA
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + Sh::STG_DBL);
  uint64_t* empty = full + 2;
  // record buffer: rec[(q*NS + j)*JS + comp*CELLS + cell], then qs[(q*QSD + x)*CELLS + cell]

  const int tid = threadIdx.x;
  const long ntiles = (E + CELLS - 1) / CELLS;
  if ((long)blockIdx.x >= ntiles) return;
  const long my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  for (int i = tid; i < Sh::TAB0; i += Sh::THREADS) smem[i] = tab[i];
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&full[b], Sh::PROD);
      mbar_init(&empty[b], Sh::ACC / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid < Sh::ACC) {
    // ---------------- consumers ----------------
    const PairSlot sl = pair_slot<Sh>(tid);
    const int lane = tid & 31;
    for (long it = 0; it < my_tiles; ++it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      const int b = (int)(it & 1);
      double a4[2][2][3][3];
      double t1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // sum_q mu' g_j.g_k
      zero_tile(a4);
      mbar_wait(&full[b], (uint32_t)((it >> 1) & 1));
      const double* rec = sRec + b * Sh::REC_DBL;
      const double* qsb = rec + Q * NS * Sh::JS;
      if (sl.active && !(PAIR_ABL & 1)) {
#pragma unroll kPairWsQUnroll
        for (int q = 0; q < Q; ++q)
          pair_point<Sh>(a4, t1, rec + q * NS * Sh::JS + sl.cell,
                         qsb + q * Sh::QSD * CELLS + sl.cell, sl.j0, sl.k0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[b]);
      // this warp's cells only: its previous bulk stores have read its staging rows
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
      add_t1(a4, t1);
      if (sl.active && !(PAIR_ABL & 16)) pair_stage<Sh>(sStg + sl.cell * Sh::CSTRIDE, a4, sl);
      if ((PAIR_ABL & 16) && sl.active) {  // keep the accumulate alive: one value per thread
        double sum = 0;
        for (int i = 0; i < 36; ++i) sum += (&a4[0][0][0][0])[i];
        sStg[sl.cell * Sh::CSTRIDE + lane % Sh::NTILE] = sum;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0 && !(PAIR_ABL & 2)) {
        const int cw = (tid >> 5) * Sh::WCELLS;
        for (int c = cw; c < min(cw + Sh::WCELLS, nt); ++c) {
          double* dst = A + (c0 + c) * (size_t)Sh::N * Sh::N;
          if (acc)
            bulk_s2g_add(dst, sStg + c * Sh::CSTRIDE, Sh::N * Sh::N * 8);
          else
            bulk_s2g(dst, sStg + c * Sh::CSTRIDE, Sh::N * Sh::N * 8);
        }
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ---------------- producers: inputs (cp.async, one tile ahead), geometry, records ----
    const int pt = tid - Sh::ACC;
    auto prefetch = [&](long it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      double* in = sIn + (it & 1) * Sh::IN_DBL;
      for (int i = pt; i < nt * 12; i += Sh::PROD) cp_async8(&in[i], coords + c0 * 12 + i);
      for (int i = pt; i < nt * Sh::NCOEF; i += Sh::PROD)
        cp_async8(&in[CELLS * 12 + (i / Sh::NCOEF) * Sh::CF + i % Sh::NCOEF], coef + c0 * Sh::NCOEF + i);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    prefetch(0);
    for (long it = 0; it < my_tiles; ++it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      const int b = (int)(it & 1);
      const double* in = sIn + b * Sh::IN_DBL;
      if (it + 1 < my_tiles) {
        prefetch(it + 1);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
      named_bar(2, Sh::PROD);
      if (pt < CELLS && !(PAIR_ABL & 8)) {
        double x[12];
#pragma unroll
        for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
          x[r] = pt < nt ? in[pt * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
        const Geo g = cell_geometry(x);
        double* cd = sCell + pt * Sh::CELLD;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) cd[a * 3 + bb] = g.K[a][bb];
        cd[9] = g.adet;
      }
      named_bar(2, Sh::PROD);
      if (it >= 2) mbar_wait(&empty[b], (uint32_t)(((it >> 1) - 1) & 1));
      double* rec = sRec + b * Sh::REC_DBL;
      double* qsb = rec + Q * NS * Sh::JS;
      // thread -> (cell, q): K, mu', lam' once, then the 10 records g_j = K^T D phi_j
      for (int task = pt; task < ((PAIR_ABL & 4) ? 0 : CELLS * Q); task += Sh::PROD) {
        // q, q + Q/2 share a half-warp: their record rows start NS*JS*Q/2 doubles apart,
        // opposite bank halves for the c3 shape (conflict-free 8-byte record stores)
        const int c = task % CELLS, r = task / CELLS;
        const int q = (Q % 2 == 0) ? (r & 1) * (Q / 2) + (r >> 1) : r;
        const double* Kp = sCell + c * Sh::CELLD;
        double K[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) K[i] = Kp[i];
        const double* cf = in + CELLS * 12 + c * Sh::CF;
        double muq = 0, lamq = 0;
        if (c < nt) {
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            muq += cf[m] * sP[q * 4 + m];
            lamq += cf[4 + m] * sP[q * 4 + m];
          }
        }
        const double wq = sW[q] * Kp[9];
        double* qs = qsb + q * Sh::QSD * CELLS + c;
        qs[0] = lamq * wq;
        qs[CELLS] = muq * wq;
        double* rr = rec + q * NS * Sh::JS + c;
#pragma unroll 5
        for (int j = 0; j < NS; ++j) {
          const double d0 = sD[(0 * Q + q) * NS + j], d1 = sD[(1 * Q + q) * NS + j],
                       d2 = sD[(2 * Q + q) * NS + j];
#pragma unroll
          for (int bb = 0; bb < 3; ++bb)
            rr[j * Sh::JS + bb * CELLS] = K[0 * 3 + bb] * d0 + K[1 * 3 + bb] * d1 + K[2 * 3 + bb] * d2;
        }
      }
      mbar_arrive_cta(&full[b]);  // release: this tile's records are visible
      named_bar(2, Sh::PROD);     // sIn[b] / sCell reused two tiles later
    }
  }
}

// ============================================================================
// St Venant-Kirchhoff: flat (all threads in every phase), 2 CTAs per SM
// ============================================================================
template <int KIND, int NS, int Q>
__global__ void __launch_bounds__(128, PAIR_FLAT_CTAS)
    pair_flat_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                     const double* __restrict__ tab, double* __restrict__ A, int acc) {
  using Sh = PairShape<KIND, NS, Q>;
  constexpr int CELLS = Sh::CELLS;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;
  double* sD = sW + Q;                      // [3][Q][NS]
  double* sP = sD + 3 * Q * NS;             // [Q][4]
  double* sCell = smem + Sh::TAB;           // [CELLS][CELLD]
  double* sIn = sCell + CELLS * Sh::CELLD;  // [CELLS][12] | [CELLS][NCOEF]
  double* sU = sIn + Sh::IN_DBL;            // records of a chunk / output staging
  double* sQs = sU + Sh::QC * NS * Sh::JS;  // [QC][QSD][CELLS]

  const int tid = threadIdx.x;
  for (int i = tid; i < Sh::TAB0; i += Sh::THREADS) smem[i] = tab[i];
  const PairSlot sl = pair_slot<Sh>(tid);

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
        for (int b = 0; b < 3; ++b) cd[a * 3 + b] = g.K[a][b];
      cd[9] = g.adet;
    }
    __syncthreads();
    double a4[2][2][3][3];
    double t1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // SVK: sum_q mu' h_j.h_k; elasticity: mu' g_j.g_k
    zero_tile(a4);
#pragma unroll 1
    for (int ch = 0; ch < Sh::NCHUNK; ++ch) {
      const int q0 = ch * Sh::QC;
      const int qn = min(Sh::QC, Q - q0);
      // ---- per (cell, q), one thread: F = I + grad w, tr E, F F^T, lam', mu',
      //      then the 10 records g_j, h_j = F g_j (F in registers)
      // warp-owned cells (JS odd): q and q + 4 share a half-warp, so the record
      // stores of its 16 lanes fall in opposite bank halves
      constexpr int NTASK = Sh::WARP_CELLS ? CELLS * ((Sh::QC + 7) / 8 * 8) : CELLS * Sh::QC;
      for (int task = tid; task < ((PAIR_ABL & 4) ? 0 : NTASK); task += Sh::THREADS) {
        const int c = task % CELLS, r = task / CELLS;
        const int ql = Sh::WARP_CELLS ? (r >> 3) * 8 + (r & 1) * 4 + ((r & 7) >> 1) : r;
        if (ql >= qn) continue;
        const int q = q0 + ql;
        pair_point_setup<Sh::SVK, NS, Q, CELLS, Sh::JS, Sh::NCOEF>(
            sCell + c * Sh::CELLD, sIn + CELLS * 12 + c * Sh::NCOEF, c < nt, q, sW, sD, sP,
            sQs + ql * Sh::QSD * CELLS + c, sU + ql * NS * Sh::JS + c);
      }
      __syncthreads();
      if (ch == Sh::NCHUNK - 1 && tile + gridDim.x < ntiles) prefetch(tile + gridDim.x);
      if (sl.active && !(PAIR_ABL & 1)) {
#pragma unroll kPairQUnroll
        for (int ql = 0; ql < qn; ++ql)
          pair_point<Sh>(a4, t1, sU + ql * NS * Sh::JS + sl.cell,
                         sQs + ql * Sh::QSD * CELLS + sl.cell, sl.j0, sl.k0);
      }
      __syncthreads();  // records consumed (next chunk / staging overwrite them)
    }
    if constexpr (Sh::SVK) svk_unfold(a4);
    add_t1(a4, t1);
    if (sl.active) pair_stage<Sh>(sU + sl.cell * Sh::CSTRIDE, a4, sl);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) pair_bulk_store<Sh>(A, c0, nt, sU, acc);
  }
  if (tid == 0) bulk_wait0();
}


// The reference tables of the SVK ring kernel as a kernel parameter (constant
// bank c[0]): the producers' table reads leave the shared-memory crossbar.
template <int NS, int Q>
struct SvkTables {
  double W[Q];
  double D[3 * Q * NS];
  double P[Q * 4];
};

// ============================================================================
// St Venant-Kirchhoff, warp-specialised: NPW producer warps run the per-point setup
// (one (cell, q) per lane: 2 points x 16 cells per ring stage) into an NSLOT-slot
// record ring while 8 consumer warps accumulate.  Consumer lane = (cell, tile): the
// warp's two (j,k) tiles are warp-uniform, so the 10 off-diagonal 2x2 tiles fill 5
// warps and the 5 diagonal ones -- whose k side is their j side (pair_point_diag:
// 20 instead of 32 loads, 87 instead of 126 FP64 instructions per point) -- 3 warps.
// With G records (PAIR_SVK_GREC) the producers store h_j and G_jk = g_j.g_k per point
// and the consumers read 24 (diagonal tiles 17) operands per point.  The tile's 16
// cells are staged together: each consumer warp stages its tiles and arrives on an
// mbarrier; one issuer bulk-stores the 16 cells and releases the staging halfway
// through the next tile, so no consumer waits for another at the tile end.  Of the
// 4 producer warps the first only loads inputs and computes the geometry, keeping
// the sub-partition with two off-diagonal consumer warps free of setup work.
// ============================================================================
template <int NS_, int Q>
struct SvkWsShape {
  static constexpr bool SVK = true;
  static constexpr int NS = NS_;
  static constexpr int N = 3 * NS;
  static constexpr int NJ = NS / 2;
  static constexpr int NTILE = NJ * (NJ + 1) / 2;
  static constexpr int CELLS = PAIR_SVK_CELLS;
  static constexpr int NPW = PAIR_SVK_PW;               // producer warps (stage g: warp g % NPW)
  static constexpr int NSLOT = PAIR_SVK_SLOTS > 0 ? PAIR_SVK_SLOTS : NPW;  // ring slots
  // consumer warps: lane = (cell, one of the warp's two tiles); the 10 off-diagonal
  // tiles in NOFFW warps, the 5 diagonal ones (k side = j side) in NDIAGW warps
  static constexpr int NOFF = NTILE - NJ;
  static constexpr int NOFFW = NOFF / 2, NDIAGW = (NJ + 1) / 2;
  static constexpr int ACC = 32 * (NOFFW + NDIAGW);
  // producer warps: 4, of which the last NPW build the ring stages (stage g: worker
  // g % NPW); with NPW = 3 the first producer warp only loads inputs and geometry, so
  // its sub-partition carries the two off-diagonal consumer warps 0 and 4
  static constexpr int NPROD_W = 4, PW0 = NPROD_W - NPW;
  static constexpr int PROD = 32 * NPROD_W, THREADS = ACC + PROD;
  static constexpr int CTAS_PER_SM = CELLS == 8 ? 2 : 1;
  static constexpr bool WARP_CELLS = true;  // pair_stage: diagonal mirror folded
  static constexpr int QS = 32 / CELLS;                 // points per ring stage
  static constexpr int NST = (Q + QS - 1) / QS;         // ring stages per tile
  static constexpr bool GREC = PAIR_SVK_GREC;
  static constexpr int RECD = GREC ? 3 : 6, QSD = 8;   // h (| g); al, be, mu' F F^T + sig
  static constexpr int JS = RECD * CELLS + 1;           // j stride of the records
  static constexpr int NP = NS * (NS + 1) / 2;          // (j <= k) pairs: G records
  static constexpr int GOFF = NS * JS;                  // per point: records | G | scalars
  static constexpr int QSOFF = GOFF + (GREC ? NP * CELLS : 0);
  static constexpr int PT_DBL = QSOFF + QSD * CELLS;
  static constexpr int STAGE_DBL = QS * PT_DBL;
  static constexpr int NCOEF = 3 * NS + 8;
  // coefficient rows padded to an odd stride: the producers' per-(cell, q) reads of
  // 16 cells' rows are conflict-free (stride 38 was 2-way)
  static constexpr int CF = NCOEF | 1;
  static constexpr int TAB0 = Q + 3 * Q * NS + 4 * Q;
  static constexpr int TAB = PAIR_SVK_PARAMTAB ? 0 : (TAB0 + 1) / 2 * 2;
  static constexpr int CELLD = 10;
  static constexpr int IN_DBL = (CELLS * (12 + CF) + 1) / 2 * 2;
  // staging: every cell of the tile at stride N*N + 2 (451 16-byte units: the 8 cells
  // of a quarter-warp's 16-byte stores hit distinct bank groups); the consumers stage
  // the whole tile, then each warp bulk-stores two cells
  static constexpr int CSTRIDE = N * N + 2;
  static constexpr int HEAD = TAB + 2 * (CELLS * CELLD + IN_DBL);  // double-buffered per tile
  static constexpr size_t SMEM = sizeof(double) * ((size_t)HEAD + NSLOT * STAGE_DBL +
                                                   CELLS * CSTRIDE) +
                                 (2 * NSLOT + 2) * sizeof(uint64_t);
  static_assert(CELLS == 16 && QS * CELLS == 32 && NOFF % 2 == 0 && NPW >= 1 && NPW <= 4,
                "lane maps");
  static_assert((ACC / 32) * 2 >= CELLS, "two cells' bulk stores per consumer warp");
  static_assert(HEAD % 2 == 0 && STAGE_DBL % 2 == 0 && CSTRIDE % 2 == 0, "16-byte aligned buffers");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// (j <= k) pair index of the G records
__host__ __device__ constexpr int svk_pair(int ns, int j, int k) {
  return j * (2 * ns - j + 1) / 2 + (k - j);
}

template <int NS, int Q>
__global__ void __launch_bounds__(SvkWsShape<NS, Q>::THREADS, SvkWsShape<NS, Q>::CTAS_PER_SM)
    pair_svk_ws_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                       const double* __restrict__ tab, double* __restrict__ A, int acc,
                       const __grid_constant__ SvkTables<NS, Q> ptab) {
  using Sh = SvkWsShape<NS, Q>;
  constexpr int CELLS = Sh::CELLS, NPW = Sh::NPW, NSLOT = Sh::NSLOT;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;
  double* sD = sW + Q;                        // [3][Q][NS]
  [[maybe_unused]] double* sP = sD + 3 * Q * NS;  // [Q][4]
  double* sCell = smem + Sh::TAB;             // [2][CELLS][CELLD]          (producers)
  double* sIn = sCell + 2 * CELLS * Sh::CELLD;  // [2][CELLS][12 | NCOEF]   (producers)
  double* sRing = smem + Sh::HEAD;            // [NSLOT][STAGE_DBL]  producers -> consumers
  double* sStg = sRing + NSLOT * Sh::STAGE_DBL;  // [CELLS][CSTRIDE]
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + CELLS * Sh::CSTRIDE);
  uint64_t* empty = full + NSLOT;
  uint64_t* staged = empty + NSLOT;  // every consumer warp has staged the tile
  uint64_t* sfree = staged + 1;      // the previous tile's bulk stores have read the staging
  // stage: rec[(ql*NS + j)*JS + comp*CELLS + cell], then qs[(ql*QSD + x)*CELLS + cell]

  const int tid = threadIdx.x;
  const long ntiles = (E + CELLS - 1) / CELLS;
  if ((long)blockIdx.x >= ntiles) return;
  const long my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  if (!PAIR_SVK_PARAMTAB)
    for (int i = tid; i < Sh::TAB0; i += Sh::THREADS) smem[i] = tab[i];
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 32);
      mbar_init(&empty[b], Sh::ACC / 32);
    }
    mbar_init(staged, Sh::ACC / 32);
    mbar_init(sfree, 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (tid < Sh::ACC) {
    // ---------------- consumers ----------------
    const int lane = tid & 31, warp = tid >> 5;
    const bool issuer = tid == 0;  // bulk-stores the tile's 16 cells
    const bool dwarp = warp >= Sh::NOFFW;  // warp-uniform: diagonal-tile warp
    PairSlot sl;
    {
      sl.cell = lane & 15;
      int t = 2 * (dwarp ? warp - Sh::NOFFW : warp) + (lane >> 4), TJ = 0, TK = 0;
      if (dwarp) {
        sl.active = t < Sh::NJ;
        TJ = TK = sl.active ? t : 0;
      } else {  // t-th off-diagonal tile (TJ < TK), row by row
        sl.active = true;
        for (int J = 0; J < Sh::NJ; ++J) {
          const int len = Sh::NJ - 1 - J;
          if (t < len) {
            TJ = J;
            TK = J + 1 + t;
            break;
          }
          t -= len;
        }
      }
      sl.j0 = 2 * TJ;
      sl.k0 = 2 * TK;
      sl.diag = dwarp;
    }
    int pidx[2][2];  // G record pairs of the tile (diagonal tile: (j0+1, j0) unused)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y) {
        const int j = sl.j0 + x, k = sl.k0 + y;
        pidx[x][y] = svk_pair(NS, min(j, k), max(j, k));
      }
    long g = 0;  // ring stage counter: slot g % NSLOT, use g / NSLOT
    for (long it = 0; it < my_tiles; ++it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      double a4[2][2][3][3];
      double t1[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // sum_q mu' h_j.h_k
      zero_tile(a4);
#pragma unroll 1
      for (int st = 0; st < Sh::NST; ++st, ++g) {
        const int b = (int)(g % NSLOT);
        mbar_wait(&full[b], (uint32_t)((g / NSLOT) & 1));
        const int nq = min(Sh::QS, Q - st * Sh::QS);
        if constexpr (Sh::GREC) {
          const double* pt = sRing + b * Sh::STAGE_DBL + sl.cell;  // point ql at ql * PT_DBL
          if (sl.active && !(PAIR_ABL & 1)) {
            if (dwarp) {
              if (nq == Sh::QS) {
#pragma unroll kSvkQUnroll
                for (int ql = 0; ql < Sh::QS; ++ql)
                  svk_point_g_diag<Sh>(a4, t1, pt + ql * Sh::PT_DBL, pt + ql * Sh::PT_DBL + Sh::GOFF,
                                       pt + ql * Sh::PT_DBL + Sh::QSOFF, sl.j0, pidx);
              } else {
                for (int ql = 0; ql < nq; ++ql)
                  svk_point_g_diag<Sh>(a4, t1, pt + ql * Sh::PT_DBL, pt + ql * Sh::PT_DBL + Sh::GOFF,
                                       pt + ql * Sh::PT_DBL + Sh::QSOFF, sl.j0, pidx);
              }
            } else {
              if (nq == Sh::QS) {
#pragma unroll kSvkQUnroll
                for (int ql = 0; ql < Sh::QS; ++ql)
                  svk_point_g<Sh>(a4, t1, pt + ql * Sh::PT_DBL, pt + ql * Sh::PT_DBL + Sh::GOFF,
                                  pt + ql * Sh::PT_DBL + Sh::QSOFF, sl.j0, sl.k0, pidx);
              } else {
                for (int ql = 0; ql < nq; ++ql)
                  svk_point_g<Sh>(a4, t1, pt + ql * Sh::PT_DBL, pt + ql * Sh::PT_DBL + Sh::GOFF,
                                  pt + ql * Sh::PT_DBL + Sh::QSOFF, sl.j0, sl.k0, pidx);
              }
            }
          }
        } else {
        const double* rec = sRing + b * Sh::STAGE_DBL + sl.cell;
        const double* qsb = sRing + b * Sh::STAGE_DBL + Sh::QS * NS * Sh::JS + sl.cell;
        if (sl.active && !(PAIR_ABL & 1)) {
          if (dwarp) {
            if (nq == Sh::QS) {
#pragma unroll
              for (int ql = 0; ql < Sh::QS; ++ql)
                pair_point_diag<Sh>(a4, t1, rec + ql * NS * Sh::JS, qsb + ql * Sh::QSD * CELLS,
                                    sl.j0);
            } else {
              for (int ql = 0; ql < nq; ++ql)
                pair_point_diag<Sh>(a4, t1, rec + ql * NS * Sh::JS, qsb + ql * Sh::QSD * CELLS,
                                    sl.j0);
            }
          } else {
            if (nq == Sh::QS) {
#pragma unroll
              for (int ql = 0; ql < Sh::QS; ++ql)
                pair_point<Sh>(a4, t1, rec + ql * NS * Sh::JS, qsb + ql * Sh::QSD * CELLS, sl.j0,
                               sl.k0);
            } else {
              for (int ql = 0; ql < nq; ++ql)
                pair_point<Sh>(a4, t1, rec + ql * NS * Sh::JS, qsb + ql * Sh::QSD * CELLS, sl.j0,
                               sl.k0);
            }
          }
        }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(&empty[b]);
        // halfway through the tile the previous tile's bulk stores have long read the
        // staging: release it (no consumer warp waits for another at the tile end)
        if (issuer && it > 0 && st == Sh::NST / 2) {
          bulk_wait_read0();
          mbar_arrive_cta(sfree);
        }
      }
      svk_unfold(a4);
      add_t1(a4, t1);
      // the tile's cells through their staging rows: every consumer warp stages its
      // tiles and arrives; the issuer bulk-stores the 16 cells once all have
      if (it > 0) mbar_wait(sfree, (uint32_t)((it - 1) & 1));
      if (sl.active) pair_stage<Sh>(sStg + sl.cell * Sh::CSTRIDE, a4, sl);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(staged);
      if (issuer) {
        mbar_wait(staged, (uint32_t)(it & 1));
        for (int cell = 0; cell < nt; ++cell) {
          double* dst = A + (c0 + cell) * (size_t)Sh::N * Sh::N;
          if (acc)
            bulk_s2g_add(dst, sStg + cell * Sh::CSTRIDE, Sh::N * Sh::N * 8);
          else
            bulk_s2g(dst, sStg + cell * Sh::CSTRIDE, Sh::N * Sh::N * 8);
        }
        bulk_commit();
      }
    }
    if (issuer) bulk_wait0();
  } else {
    // ---------------- producer warps: inputs (cp.async, one tile ahead), geometry,
    //                  per-point setup; warp pw takes stages g = pw mod NPW ----------------
    const int ptid = tid - Sh::ACC, pt = ptid & 31, pw = ptid >> 5;
    auto prefetch = [&](long it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      double* in = sIn + (it & 1) * Sh::IN_DBL;
      for (int i = ptid; i < nt * 12; i += Sh::PROD) cp_async8(&in[i], coords + c0 * 12 + i);
      for (int i = ptid; i < nt * Sh::NCOEF; i += Sh::PROD)
        cp_async8(&in[CELLS * 12 + (i / Sh::NCOEF) * Sh::CF + i % Sh::NCOEF],
                  coef + c0 * Sh::NCOEF + i);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    prefetch(0);
    const int c = pt % CELLS, ql = pt / CELLS;
    long g = 0;
    for (long it = 0; it < my_tiles; ++it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      const double* in = sIn + (it & 1) * Sh::IN_DBL;
      double* cell = sCell + (it & 1) * CELLS * Sh::CELLD;
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      named_bar(1, Sh::PROD);  // this tile's inputs have landed (all producer threads' copies)
      if (ptid < CELLS) {
        double x[12];
#pragma unroll
        for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
          x[r] = ptid < nt ? in[ptid * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
        const Geo geo = cell_geometry(x);
        double* cd = cell + ptid * Sh::CELLD;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) cd[a * 3 + bb] = geo.K[a][bb];
        cd[9] = geo.adet;
      }
      // geometry visible; every producer is past the previous tile, whose input buffer
      // the next prefetch overwrites
      named_bar(1, Sh::PROD);
      if (it + 1 < my_tiles) prefetch(it + 1);
#pragma unroll 1
      for (int st = 0; st < Sh::NST; ++st, ++g) {
        if ((int)(g % NPW) != pw - Sh::PW0) continue;  // helper warps (pw < PW0): none
        const int b = (int)(g % NSLOT);
        if (g >= NSLOT) mbar_wait(&empty[b], (uint32_t)((g / NSLOT - 1) & 1));
        double* rec = sRing + b * Sh::STAGE_DBL;
        const int q = st * Sh::QS + ql;
        if (q < Q && !(PAIR_ABL & 4) && Sh::GREC) {
          double* pp = rec + ql * Sh::PT_DBL + c;
          const double* Kc = cell + c * Sh::CELLD;
          const double* cf = in + CELLS * 12 + c * Sh::CF;
          if constexpr (PAIR_SVK_PARAMTAB)
            svk_setup_g<NS, Q, CELLS, Sh::JS>(Kc, cf, c < nt, q, ptab.W, ptab.D, ptab.P,
                                             pp + Sh::QSOFF, pp, pp + Sh::GOFF);
          else
            svk_setup_g<NS, Q, CELLS, Sh::JS>(Kc, cf, c < nt, q, sW, sD, sP, pp + Sh::QSOFF, pp,
                                             pp + Sh::GOFF);
        } else if (q < Q && !(PAIR_ABL & 4)) {
          double* qsp = rec + Sh::QS * NS * Sh::JS + ql * Sh::QSD * CELLS + c;
          double* rp = rec + ql * NS * Sh::JS + c;
          const double* Kc = cell + c * Sh::CELLD;
          const double* cf = in + CELLS * 12 + c * Sh::CF;
          if constexpr (PAIR_SVK_PARAMTAB)
            pair_point_setup<true, NS, Q, CELLS, Sh::JS, Sh::NCOEF>(Kc, cf, c < nt, q, ptab.W,
                                                                   ptab.D, ptab.P, qsp, rp);
          else
            pair_point_setup<true, NS, Q, CELLS, Sh::JS, Sh::NCOEF>(Kc, cf, c < nt, q, sW, sD, sP,
                                                                   qsp, rp);
        }
        mbar_arrive_cta(&full[b]);  // release: this stage's records are visible
      }
    }
  }
}

template <int NS, int Q>
static cudaError_t launch_svk_ws(long E, const double* coords, const double* coef,
                                 const double* tab, const double* htab, double* A, int acc,
                                 cudaStream_t s) {
  using Sh = SvkWsShape<NS, Q>;
  SvkTables<NS, Q> pt;  // W | D | P, the layout of tab (host copy)
  static_assert(sizeof(pt) == sizeof(double) * Sh::TAB0, "table layout");
  if (htab) std::memcpy(&pt, htab, sizeof pt);
  else if (PAIR_SVK_PARAMTAB) return cudaErrorInvalidValue;
  auto kern = pair_svk_ws_kernel<NS, Q>;
  static const char once_key = 0;  // one per (kernel instantiation, device)
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    if (e != cudaSuccess) return e;
    return cudaSuccess;
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  const long maxc = (long)Sh::CTAS_PER_SM * num_sms();
  const int grid = (int)(ntiles < maxc ? ntiles : maxc);
  kern<<<grid, Sh::THREADS, Sh::SMEM, s>>>(E, coords, coef, tab, A, acc, pt);
  return cudaGetLastError();
}

template <int KIND, int NS, int Q>
static cudaError_t launch_pair_t(long E, const double* coords, const double* coef,
                                 const double* tab, const double* htab, double* A, int acc,
                                 cudaStream_t s) {
  using Sh = PairShape<KIND, NS, Q>;
  if constexpr (Sh::SVK && PAIR_SVK_WS)
    return launch_svk_ws<NS, Q>(E, coords, coef, tab, htab, A, acc, s);
  auto kern = (Sh::SVK || Sh::FLAT) ? pair_flat_kernel<KIND, NS, Q> : pair_ws_kernel<NS, Q>;
  static const char once_key = 0;  // one per (kernel instantiation, device)
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    if (e != cudaSuccess) return e;
    return cudaSuccess;
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  const long maxc = (long)Sh::CTAS_PER_SM * num_sms();
  const int grid = (int)(ntiles < maxc ? ntiles : maxc);
  kern<<<grid, Sh::THREADS, Sh::SMEM, s>>>(E, coords, coef, tab, A, acc);
  return cudaGetLastError();
}

bool pair_supported(int kind, int nq, int ns) {
  if (ns != 10) return false;
  if (kind == FEMGPU_ELASTICITY) return nq == 8 || nq == 27;
  if (kind == FEMGPU_HYPERELASTICITY) return nq == 27 || nq == 8;
  return false;
}

cudaError_t launch_pair(int kind, int nq, int ns, long E, const double* coords, const double* coef,
                        const double* tab, const double* htab, double* A, int acc,
                        cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  if (ns == 10) {
    if (kind == FEMGPU_ELASTICITY && nq == 8)
      return launch_pair_t<FEMGPU_ELASTICITY, 10, 8>(E, coords, coef, tab, htab, A, acc, s);
    if (kind == FEMGPU_ELASTICITY && nq == 27)
      return launch_pair_t<FEMGPU_ELASTICITY, 10, 27>(E, coords, coef, tab, htab, A, acc, s);
    if (kind == FEMGPU_HYPERELASTICITY && nq == 27)
      return launch_pair_t<FEMGPU_HYPERELASTICITY, 10, 27>(E, coords, coef, tab, htab, A, acc, s);
    if (kind == FEMGPU_HYPERELASTICITY && nq == 8)
      return launch_pair_t<FEMGPU_HYPERELASTICITY, 10, 8>(E, coords, coef, tab, htab, A, acc, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
