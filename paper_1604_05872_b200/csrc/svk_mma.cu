// svk_mma.cu -- St Venant-Kirchhoff Jacobian (config 4) on the FP64 tensor cores.
//
// Same schedule as femopt's QUADRATURE plan for this form (sum over quadrature points
// with the per-point operands hoisted, proj/src/sharing.cpp:409-607), but the
// contraction over q is cut into three dense products per cell that the DMMA pipe
// runs, instead of per-pair FMA streams on the CUDA cores (pair.cu):
//
//   A_e[(c,j),(d,k)] = sum_q lam' h_j[c] h_k[d] + mu' h_k[c] h_j[d]
//                      + m_cd(q) G_jk(q) + d_cd mu' h_j.h_k
//   with h_j = F g_j, G_jk = g_j.g_k, m_cd = mu' (F F^T)_cd + d_cd sig,
//   sig = w'(lam tr E - mu)   (pair.cu header: the stress term s_j.g_k of the
//   linearised SVK form is sig g_j.g_k + mu' h_j.h_k).
//
// With X_q the 30-vector X_q[(c,j)] = h_j[c] (row r = 10 c + j, the element
// matrix's own row order):
//   Ylam = sum_q lam'_q X_q X_q^T,  Ymu = sum_q mu'_q X_q X_q^T   (30 x 30, K = Q)
//   W[cd, p] = sum_q m_cd(q) G_p(q)                               (6 x 55,  K = Q)
// and then   A[(c,j),(d,k)] = Ylam[(c,j),(d,k)] + Ymu[(c,k),(d,j)] + W[cd, jk]
//                              + d_cd sum_e Ymu[(e,j),(e,k)].
// The swap term mu' h_k[c] h_j[d] is Ymu read at permuted indices, and its trace
// gives the mu' h_j.h_k part of the stress term, so the two symmetric rank-1
// updates per point carry every h-dependent term.
//
// Kernel (one CTA of 12 warps per SM, persistent over 8-cell tiles):
//  * 4 producer warps: one (cell, point) per lane, 8 cells x 4 points per ring stage
//    (one k4 step of the products): F = I + grad w, tr E, m_cd, lam', mu', the
//    records g_j = K^T D phi_j, X = F g_j and the 55 G_jk; stored in the DMMA
//    fragment order of mma.m8n8k4 (cell stride == 4 mod 16 doubles: conflict-free
//    record stores; every fragment load is 32 consecutive doubles);
//  * 8 consumer warps, one cell each: per stage 10 + 10 DMMA for the upper 8x8 tiles
//    of Ylam and Ymu (32 x 32 padded; a symmetric product reuses one fragment as A of
//    the row tile and B of the column tile) and 7 for W (8 x 56 padded); the
//    accumulators stay in registers for the cell's Q points; then Ymu and W go to
//    the warp's scratch, each lane finishes its Ylam entries (permuted Ymu, W, trace),
//    stages the symmetric element matrix and one TMA bulk copy writes it.
//
// Measured on c4 (one B200): 1.431 ms against 1.107 ms for the DFMA
// pair kernel, so AUTO ranks this schedule second.  Ablations (SVKM_ABL): the DMMA
// products alone run 0.676 ms (76 % of the DMMA peak on 96.8 k flops/cell); with
// the producers 0.966 ms; the assembly adds 0.47 ms (all consumer warps run it at
// once while the DMMA pipe idles).
#include "common.cuh"
#include "femgpu_internal.h"
#include "../../include/femgpu.h"

#ifndef SVKM_ABL  // development ablations: bit 0 no DMMA, bit 1 no producer setup, bit 2 no assembly
#define SVKM_ABL 0
#endif
#ifndef SVKM_CELLS
#define SVKM_CELLS 8  // cells per CTA tile (one consumer warp each): 8 -> one CTA per SM,
                      // 4 -> two independent CTAs per SM with 8-point stages (measured
                      // 1.476 vs 1.431 ms on c4: the two rings couple worse to the producers)
#endif
#ifndef SVKM_SLOTS
#define SVKM_SLOTS (SVKM_CELLS == 8 ? 4 : 2)  // ring stages in flight
#endif

namespace femgpu {
namespace {

template <int Q_>
struct SvkMmaShape {
  static constexpr int Q = Q_;
  static constexpr int NS = 10, N = 30;
  static constexpr int CELLS = SVKM_CELLS;  // cells per CTA tile: consumer warp w owns cell w
  static constexpr int CTAS_PER_SM = 8 / CELLS;
  static constexpr int QS = 32 / CELLS;      // points per ring stage (one producer lane each)
  static constexpr int KSPS = QS / 4;        // k4 steps per stage
  static constexpr int NST = (Q + QS - 1) / QS;
  static constexpr int NPW = CELLS / 2;      // producer warps; stage g is built by warp g % NPW
  static constexpr int NSLOT = SVKM_SLOTS;
  static constexpr int ACC = 32 * CELLS, PROD = 32 * NPW, THREADS = ACC + PROD;
  static constexpr int NP = NS * (NS + 1) / 2;  // 55 (j <= k) pairs
  static constexpr int NPT = (NP + 7) / 8;       // 7 column tiles of W
  static constexpr int NYT = 10;                  // upper 8x8 tiles of a 32x32 product
  // per cell and k4 step: X [4 row tiles][32] | G [NPT][32] | M [32] | lam', mu' [4][2]
  static constexpr int OX = 0, OG = 4 * 32, OM = OG + NPT * 32, OLM = OM + 32;
  static constexpr int KB0 = OLM + 8;
  static constexpr int KB = KB0 + ((4 - KB0 % 16) + 16) % 16;  // == 4 mod 16
  // per cell: KSPS k4 blocks (== 4 resp. 8 mod 16: the producer lanes (cell, point) of a
  // half-warp store to 16 distinct banks)
  static constexpr int CS = KSPS * KB;
  static constexpr int STAGE_DBL = CELLS * CS;
  // consumer scratch per warp: Ymu [32][YS] | W [8][56]; the staged element matrix
  // (N*N) aliases it once the scratch has been read
  static constexpr int YS = 34;
  static constexpr int OW = 32 * YS;
  static constexpr int SCR = OW + 8 * NPT * 8;
  static constexpr int NCOEF = 3 * NS + 8;
  static constexpr int CF = NCOEF | 1;  // odd coefficient-row stride (conflict-free reads)
  static constexpr int TAB0 = Q + 3 * Q * NS + 4 * Q;  // W | D | P
  static constexpr int TAB = (TAB0 + 1) / 2 * 2;
  static constexpr int CELLD = 10;      // K (9), |det J|
  static constexpr int IN_DBL = (CELLS * (12 + CF) + 1) / 2 * 2;
  static constexpr int HEAD = TAB + 2 * (CELLS * CELLD + IN_DBL);
  static constexpr size_t SMEM =
      sizeof(double) * ((size_t)HEAD + NSLOT * STAGE_DBL + CELLS * SCR) +
      2 * NSLOT * sizeof(uint64_t);
  static_assert(KB % 16 == 4 && CS % 16 == 4 * KSPS && STAGE_DBL % 2 == 0 && HEAD % 2 == 0 &&
                    SCR % 2 == 0 && QS % 4 == 0 && NSLOT % NPW == 0,
                "aligned, conflict-free stage layout; a producer warp owns its ring slots");
  static_assert(SCR >= N * N, "staging fits the scratch");
  static_assert(SMEM * CTAS_PER_SM <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ void dmma8x8x4(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_named(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// upper 8x8 tile t (0..9) of a 4x4 tile grid -> (row tile, column tile)
__host__ __device__ constexpr int ytile_m(int t) { return t < 4 ? 0 : t < 7 ? 1 : t < 9 ? 2 : 3; }
__host__ __device__ constexpr int ytile_n(int t) {
  return t < 4 ? t : t < 7 ? t - 3 : t < 9 ? t - 5 : 3;
}
// (j <= k) pair index
__device__ __forceinline__ int pair_idx(int j, int k) { return j * 10 - j * (j - 1) / 2 + (k - j); }
// (c <= d) component-pair index: 00 01 02 11 12 22
__device__ __forceinline__ int cd_idx(int c, int d) { return c == 0 ? d : c == 1 ? 2 + d : 5; }

template <int Q>
__global__ void __launch_bounds__(SvkMmaShape<Q>::THREADS, SvkMmaShape<Q>::CTAS_PER_SM)
    svk_mma_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                   const double* __restrict__ tab, double* __restrict__ A, int acc) {
  using Sh = SvkMmaShape<Q>;
  constexpr int CELLS = Sh::CELLS, NS = Sh::NS, NSLOT = Sh::NSLOT;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem;
  double* sD = sW + Q;                          // [3][Q][NS]
  double* sP = sD + 3 * Q * NS;                 // [Q][4]
  double* sCell = smem + Sh::TAB;               // [2][CELLS][CELLD]
  double* sIn = sCell + 2 * CELLS * Sh::CELLD;  // [2][CELLS][12 | CF]
  double* sRing = smem + Sh::HEAD;              // [NSLOT][STAGE_DBL]
  double* sScr = sRing + NSLOT * Sh::STAGE_DBL; // [CELLS][SCR]
  uint64_t* full = reinterpret_cast<uint64_t*>(sScr + CELLS * Sh::SCR);
  uint64_t* empty = full + NSLOT;

  const int tid = threadIdx.x;
  const long ntiles = (E + CELLS - 1) / CELLS;
  if ((long)blockIdx.x >= ntiles) return;
  const long my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  for (int i = tid; i < Sh::TAB0; i += Sh::THREADS) smem[i] = tab[i];
  if (tid == 0) {
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&full[b], 32);
      mbar_init(&empty[b], CELLS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid < Sh::ACC) {
    // ---------------- consumers: warp w = cell w of each tile ----------------
    const int lane = tid & 31, w = tid >> 5;
    const int qi = lane & 3, gi = lane >> 2;
    double* scr = sScr + w * Sh::SCR;
    long g = 0;
    for (long it = 0; it < my_tiles; ++it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      double yl[Sh::NYT][2], ym[Sh::NYT][2], wc[Sh::NPT][2];
#pragma unroll
      for (int t = 0; t < Sh::NYT; ++t) yl[t][0] = yl[t][1] = ym[t][0] = ym[t][1] = 0.0;
#pragma unroll
      for (int t = 0; t < Sh::NPT; ++t) wc[t][0] = wc[t][1] = 0.0;
#pragma unroll 1
      for (int st = 0; st < Sh::NST; ++st, ++g) {
        const int b = (int)(g % NSLOT);
        mbar_wait(&full[b], (uint32_t)((g / NSLOT) & 1));
        const int nks = min(Sh::KSPS, (Q - st * Sh::QS + 3) / 4);
#pragma unroll 1
        for (int ks = 0; ks < nks; ++ks) {
          const double* sg = sRing + b * Sh::STAGE_DBL + w * Sh::CS + ks * Sh::KB;
          const double lam = sg[Sh::OLM + 2 * qi], mu = sg[Sh::OLM + 2 * qi + 1];
          double x[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) x[m] = sg[Sh::OX + 32 * m + lane];
          const double mf = sg[Sh::OM + lane];
          if (!(SVKM_ABL & 1)) {
#pragma unroll
            for (int t = 0; t < Sh::NPT; ++t) dmma8x8x4(wc[t], mf, sg[Sh::OG + 32 * t + lane]);
#pragma unroll
            for (int t = 0; t < Sh::NYT; ++t) {
              dmma8x8x4(yl[t], lam * x[ytile_m(t)], x[ytile_n(t)]);
              dmma8x8x4(ym[t], mu * x[ytile_m(t)], x[ytile_n(t)]);
            }
          } else {  // ablation: keep the loads alive
            yl[0][0] += lam * x[0] + mf + x[1] + x[2] + x[3];
            ym[0][0] += mu;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);
      }
      // ---- assembly: Ymu and W through the scratch, then the element matrix ----
      if (lane == 0) bulk_wait_read0();  // the previous tile's bulk store has read it
      __syncwarp();
      if (SVKM_ABL & 4) {
        double v = 0;
#pragma unroll
        for (int t = 0; t < Sh::NYT; ++t) v += yl[t][0] + yl[t][1] + ym[t][0] + ym[t][1];
#pragma unroll
        for (int t = 0; t < Sh::NPT; ++t) v += wc[t][0] + wc[t][1];
        scr[lane] = v;
      } else {
#pragma unroll
      for (int t = 0; t < Sh::NYT; ++t) {
        const int r = 8 * ytile_m(t) + gi, s = 8 * ytile_n(t) + 2 * qi;
        *reinterpret_cast<double2*>(&scr[r * Sh::YS + s]) = make_double2(ym[t][0], ym[t][1]);
      }
#pragma unroll
      for (int t = 0; t < Sh::NPT; ++t)
        *reinterpret_cast<double2*>(&scr[Sh::OW + gi * (8 * Sh::NPT) + 8 * t + 2 * qi]) =
            make_double2(wc[t][0], wc[t][1]);
      __syncwarp();
      double av[Sh::NYT][2];
#pragma unroll
      for (int t = 0; t < Sh::NYT; ++t)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = 8 * ytile_m(t) + gi, s = 8 * ytile_n(t) + 2 * qi + i;
          double v = 0.0;
          if (r <= s && s < Sh::N) {
            const int c = r / 10, j = r - 10 * c, d = s / 10, k = s - 10 * d;
            // swap term: Ymu[(c,k),(d,j)], from the stored upper triangle
            const double ymu = c == d ? scr[r * Sh::YS + s] : scr[(10 * c + k) * Sh::YS + 10 * d + j];
            v = yl[t][i] + ymu +
                scr[Sh::OW + cd_idx(c, d) * (8 * Sh::NPT) + pair_idx(min(j, k), max(j, k))];
            if (c == d)
              v += scr[j * Sh::YS + k] + scr[(10 + j) * Sh::YS + 10 + k] +
                   scr[(20 + j) * Sh::YS + 20 + k];
          }
          av[t][i] = v;
        }
      __syncwarp();  // scratch read: it becomes the staging
#pragma unroll
      for (int t = 0; t < Sh::NYT; ++t)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = 8 * ytile_m(t) + gi, s = 8 * ytile_n(t) + 2 * qi + i;
          if (r <= s && s < Sh::N) {
            scr[r * Sh::N + s] = av[t][i];
            if (r != s) scr[s * Sh::N + r] = av[t][i];
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0 && w < nt) {
        double* dst = A + (c0 + w) * (size_t)(Sh::N * Sh::N);
        if (acc)
          bulk_s2g_add(dst, scr, Sh::N * Sh::N * 8);
        else
          bulk_s2g(dst, scr, Sh::N * Sh::N * 8);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    // ---------------- producers ----------------
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
    const int c = pt / Sh::QS, qq = pt % Sh::QS;  // (cell, point of the stage)
    const int ql = qq & 3;                           // point within its k4 step
    long g = 0;
    for (long it = 0; it < my_tiles; ++it) {
      const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
      const int nt = (int)min((long)CELLS, E - c0);
      const double* in = sIn + (it & 1) * Sh::IN_DBL;
      double* cell = sCell + (it & 1) * CELLS * Sh::CELLD;
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      bar_named(1, Sh::PROD);  // this tile's inputs have landed
      if (ptid < CELLS) {
        double xv[12];
#pragma unroll
        for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
          xv[r] = ptid < nt ? in[ptid * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
        const Geo geo = cell_geometry(xv);
        double* cd = cell + ptid * Sh::CELLD;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) cd[a * 3 + bb] = geo.K[a][bb];
        cd[9] = geo.adet;
      }
      bar_named(1, Sh::PROD);  // geometry visible; the previous input buffer is free
      if (it + 1 < my_tiles) prefetch(it + 1);
#pragma unroll 1
      for (int st = 0; st < Sh::NST; ++st, ++g) {
        if ((int)(g % Sh::NPW) != pw) continue;
        const int b = (int)(g % NSLOT);
        if (g >= NSLOT) mbar_wait(&empty[b], (uint32_t)((g / NSLOT - 1) & 1));
        double* sg = sRing + b * Sh::STAGE_DBL + c * Sh::CS + (qq >> 2) * Sh::KB;
        const int q = st * Sh::QS + qq;
        if (SVKM_ABL & 2) {
        } else if (q < Q) {
          const double* Kc = cell + c * Sh::CELLD;
          const double* cf = in + CELLS * 12 + c * Sh::CF;
          const bool valid = c < nt;
          auto cv = [&](int r) -> double { return valid ? cf[r] : 0.0; };
          double muq = 0, lamq = 0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            muq += cv(3 * NS + m) * sP[q * 4 + m];
            lamq += cv(3 * NS + 4 + m) * sP[q * 4 + m];
          }
          const double wq = sW[q] * Kc[9];
          double K[9];
#pragma unroll
          for (int i = 0; i < 9; ++i) K[i] = Kc[i];
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
            for (int bb = 0; bb < 3; ++bb)
              F[cc][bb] = (cc == bb ? 1.0 : 0.0) + gr[0] * K[0 * 3 + bb] + gr[1] * K[1 * 3 + bb] +
                          gr[2] * K[2 * 3 + bb];
          }
          double trE = 0.0;
#pragma unroll
          for (int a = 0; a < 3; ++a)
            trE += 0.5 * ((F[0][a] * F[0][a] + F[1][a] * F[1][a] + F[2][a] * F[2][a]) - 1.0);
          const double mw = muq * wq, sig = wq * (lamq * trE - muq);
          // m_cd = mu' (F F^T)_cd + d_cd sig, rows 00 01 02 11 12 22 (6, 7: zero)
          double* M = sg + Sh::OM + ql;
          M[0 * 4] = mw * (F[0][0] * F[0][0] + F[0][1] * F[0][1] + F[0][2] * F[0][2]) + sig;
          M[1 * 4] = mw * (F[0][0] * F[1][0] + F[0][1] * F[1][1] + F[0][2] * F[1][2]);
          M[2 * 4] = mw * (F[0][0] * F[2][0] + F[0][1] * F[2][1] + F[0][2] * F[2][2]);
          M[3 * 4] = mw * (F[1][0] * F[1][0] + F[1][1] * F[1][1] + F[1][2] * F[1][2]) + sig;
          M[4 * 4] = mw * (F[1][0] * F[2][0] + F[1][1] * F[2][1] + F[1][2] * F[2][2]);
          M[5 * 4] = mw * (F[2][0] * F[2][0] + F[2][1] * F[2][1] + F[2][2] * F[2][2]) + sig;
          M[6 * 4] = 0.0;
          M[7 * 4] = 0.0;
          sg[Sh::OLM + 2 * ql] = lamq * wq;
          sg[Sh::OLM + 2 * ql + 1] = mw;
          // g_j = K^T D phi_j; X[(c,j)] = (F g_j)[c]: row r -> X tile r/8, lane 4 (r%8) + ql
          double gv[NS][3];
#pragma unroll
          for (int j = 0; j < NS; ++j) {
#pragma unroll
            for (int bb = 0; bb < 3; ++bb)
              gv[j][bb] = K[0 * 3 + bb] * dq[0][j] + K[1 * 3 + bb] * dq[1][j] + K[2 * 3 + bb] * dq[2][j];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              const int r = 10 * a + j;
              sg[Sh::OX + 32 * (r >> 3) + 4 * (r & 7) + ql] =
                  F[a][0] * gv[j][0] + F[a][1] * gv[j][1] + F[a][2] * gv[j][2];
            }
          }
          sg[Sh::OX + 32 * 3 + 4 * 6 + ql] = 0.0;  // rows 30, 31
          sg[Sh::OX + 32 * 3 + 4 * 7 + ql] = 0.0;
          // G_p = g_j . g_k, p = (j <= k) pair: column tile p/8, lane 4 (p%8) + ql
          int p = 0;
#pragma unroll
          for (int j = 0; j < NS; ++j)
#pragma unroll
            for (int k = j; k < NS; ++k, ++p)
              sg[Sh::OG + 32 * (p >> 3) + 4 * (p & 7) + ql] =
                  gv[j][0] * gv[k][0] + gv[j][1] * gv[k][1] + gv[j][2] * gv[k][2];
#pragma unroll
          for (; p < 8 * Sh::NPT; ++p) sg[Sh::OG + 32 * (p >> 3) + 4 * (p & 7) + ql] = 0.0;
        } else {  // padding point of the last stage
#pragma unroll 4
          for (int i = 0; i < 32 * (4 + Sh::NPT + 1) / 4; ++i) sg[4 * i + ql] = 0.0;
          sg[Sh::OLM + 2 * ql] = 0.0;
          sg[Sh::OLM + 2 * ql + 1] = 0.0;
        }
        mbar_arrive(&full[b]);  // release: this stage's records are visible
      }
    }
  }
}

template <int Q>
cudaError_t launch_q(long E, const double* coords, const double* coef, const double* tab,
                     double* A, int acc, cudaStream_t s) {
  using Sh = SvkMmaShape<Q>;
  auto kern = svk_mma_kernel<Q>;
  static const char once_key = 0;
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  const long maxc = (long)Sh::CTAS_PER_SM * num_sms();
  const int grid = (int)(ntiles < maxc ? ntiles : maxc);
  kern<<<grid, Sh::THREADS, Sh::SMEM, s>>>(E, coords, coef, tab, A, acc);
  return cudaGetLastError();
}

}  // namespace

bool svk_mma_supported(int nq, int ns) { return ns == 10 && (nq == 27 || nq == 8); }

cudaError_t launch_svk_mma(int nq, int ns, long E, const double* coords, const double* coef,
                           const double* tab, double* A, int acc, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  if (ns == 10 && nq == 27) return launch_q<27>(E, coords, coef, tab, A, acc, s);
  if (ns == 10 && nq == 8) return launch_q<8>(E, coords, coef, tab, A, acc, s);
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
