// elasticity.cu -- linear elasticity element kernel on the FP64 tensor cores
// (BASELINE config 3: vector P2, P1 mu/lambda).
//
//   a(u,v) = int 2 mu eps(u):eps(v) + lam div u div v
//   A_{(c,j),(d,k)} = sum_q mu'(q) (g_j[d] g_k[c] + d_cd g_j.g_k) + lam'(q) g_j[c] g_k[d]
//   g_j[b] = sum_a K_ab D_a phi_j,  mu'(q) = W_q |det| sum_m mu_m P_m(q)  (same for lam')
//
// TENSOR schedule (femopt's pre-evaluation, preeval.cpp:279-451, applied to the
// whole form -- femopt's own plan for this form is the quadrature one, see
// SURVEY.md §8a a5): with kappa = (m, a, a') (4 x 3 x 3 = 36)
//   A^{cd}_{jk} = sum_kappa alpha^{cd}_kappa T_{kappa, jk}
//   T_{kappa,jk} = sum_q W_q P_m(q) D_a phi_j(q) D_a' phi_k(q)            (host, once)
//   alpha^{cd}_kappa = |det| (lam_m K_ac K_a'd + mu_m K_ad K_a'c + d_cd mu_m (K K^T)_aa')
// The same quadrature sum as the reference, re-associated: exact up to rounding.
// A is symmetric (alpha^{dc}_{(m,a',a)} = alpha^{cd}_{(m,a,a')}): the kernel
// computes the three off-diagonal (c<d) blocks in full and the diagonal
// blocks' upper halves, and mirrors.
//
// Tiling: the MMA rows are (cell, block) pairs -- 5 cells x 3 blocks = 15 of 16
// rows -- so one m16 tile covers all three off-diagonal blocks (0,1) (0,2)
// (1,2) of five cells (one GEMM, K = 36), and a second one their diagonal
// blocks.  A 5-cell tile's element matrices (36 KB) are contiguous in HBM:
// staged whole in shared memory and written by ONE bulk copy
// (cp.async.bulk; cp.reduce.async.bulk .add.f64 for the += contract).
//  * 7 compute warps x 3 n8 tiles: the 13 tiles of a full 10x10 block (flat
//    p = 10j + k) and the 8 of a diagonal block's upper half (rows padded to
//    even k); each warp's T fragments (27 doubles/lane) stay in registers;
//  * warp 7 (producer) bulk-copies the next tile's inputs, computes geometry
//    and alpha into double-buffered fragment tiles (named-barrier handoff);
//  * two CTAs per SM, double-buffered staging: one CTA's epilogue overlaps
//    the other's tensor-core phase, the TMA unit drains the previous tile.
// HBM-bound in principle: 7,200 B of element matrix per cell against ~34 k DMMA
// flops.  Measured (c3, profiles/): 1.68 ms vs 1.24 ms for the CUDA-core pair
// kernel -- the GEMMs alone hide behind the stores (0.94 ms), but the mirrored
// scalar slab writes of the symmetric half cost more than the DFMA work they
// replace.  So, as femopt's cost model does for this form, AUTO picks the
// quadrature schedule (pair.cu); this kernel serves SCHED_TENSOR requests.
#include <vector>

#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

namespace et {
constexpr int NS = 10;
constexpr int N = 30;
constexpr int KD = 36;                     // kappa = (m, a, a')
constexpr int KS = KD / 4;                 // k4 steps
constexpr int NF = 13;                     // n8 tiles of a full 10x10 block (104 slots)
constexpr int NSYM = 8;                    // n8 tiles of a diagonal block's padded upper half
constexpr int CELLS = 5;                   // rows (cell, block): 15 of 16
constexpr int CWARPS = 7;                  // compute warps, 3 n8 tiles each
constexpr int TPW = 3;
constexpr int PRODUCER = 7;
constexpr int WARPS = 8;
constexpr int THREADS = 32 * WARPS;
constexpr int CTHREADS = 32 * CWARPS;
constexpr int CTAS_PER_SM = 2;
constexpr int NCOEF = 8;                   // mu (P1) | lam (P1)
constexpr int STG_DBL = CELLS * N * N;     // one tile's element matrices
constexpr int AF_DBL = 2 * KS * 64;        // alpha fragments: off-diagonal | diagonal GEMM
constexpr int IN_DBL = CELLS * (12 + NCOEF) + 4;  // one input tile
constexpr int NIN = 4;                     // input ring: loads run 3 tiles ahead
constexpr int CELLD = 10;
constexpr int TF_DBL = (NF + NSYM) * KS * 32;  // T fragments (global)
constexpr size_t SMEM =
    sizeof(double) * (size_t)(2 * STG_DBL + 2 * AF_DBL + NIN * IN_DBL + CELLS * CELLD) +
    8 * NIN;
constexpr int BAR_FULL = 2;                // + buffer: alpha fragments ready
constexpr int BAR_EMPTY = 4;               // + buffer: alpha fragments consumed
constexpr int BAR_C = 1;                   // compute warps
static_assert(CWARPS * TPW == NF + NSYM, "three n8 tiles per compute warp");
}  // namespace et

// diagonal-block upper half, rows padded to even k: slot s -> j * 16 + k (-1 = pad)
__constant__ signed char c_et_sym[64][2];

namespace {
void et_sym_table(signed char (*tab)[2]) {
  int s = 0;
  for (int j = 0; j < et::NS; ++j)
    for (int k = j & ~1; k < et::NS; ++k, ++s) {
      tab[s][0] = (signed char)j;
      tab[s][1] = (signed char)k;
    }
  for (; s < 64; ++s) tab[s][0] = tab[s][1] = -1;
}
}  // namespace

__device__ __forceinline__ void et_dmma(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ void et_nbar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void et_nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
}

#ifdef ET_TRACE
__device__ unsigned long long et_trace[256][8];
#define ET_MARK(it, slot, cond) \
  if (blockIdx.x == 0 && (cond) && (it) < 256) et_trace[it][slot] = clock64()
extern "C" int femgpu_debug_trace_et(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, et_trace, sizeof(et_trace));
}
#else
#define ET_MARK(it, slot, cond)
#endif

__global__ void __launch_bounds__(et::THREADS, et::CTAS_PER_SM)
    elas_tensor_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                       const double* __restrict__ tab, double* __restrict__ A, int acc) {
  using namespace et;
  extern __shared__ __align__(1024) double smem[];
  double* sStg = smem;                    // [2][CELLS][30][30]
  double* sAF = sStg + 2 * STG_DBL;       // [2][2 gemms][KS][32][2]
  double* sIn = sAF + 2 * AF_DBL;         // [NIN][CELLS][12] | [CELLS][8]
  double* sCell = sIn + NIN * IN_DBL;     // [CELLS][10]
  uint64_t* inBar = reinterpret_cast<uint64_t*>(sCell + CELLS * CELLD);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long ntiles = (E + CELLS - 1) / CELLS;
  const long my_tiles =
      (long)blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int i = 0; i < NIN; ++i) mbar_init(&inBar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == PRODUCER) {
    // ===================== producer: inputs -> alpha fragments =====================
    auto load = [&](long it) {  // tile it -> input buffer it % NIN
      if (lane == 0 && it < my_tiles) {
        const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
        const int nt = (int)min((long)CELLS, E - c0);
        double* in = sIn + (it % NIN) * IN_DBL;
        uint64_t* bar = &inBar[it % NIN];
        mbar_expect_tx(bar, nt * (12 + NCOEF) * 8);
        bulk_g2s(in, coords + c0 * 12, nt * 12 * 8, bar);
        bulk_g2s(in + CELLS * 12 + 4, coef + c0 * NCOEF, nt * NCOEF * 8, bar);
      }
    };
    for (int i = 0; i < NIN; ++i) load(i);
    for (long it = 0; it < my_tiles; ++it) {
      const long tile = blockIdx.x + it * gridDim.x;
      const int nt = (int)min((long)CELLS, E - tile * CELLS);
      const int b = (int)(it & 1);
      double* AF = sAF + b * AF_DBL;
      const double* in = sIn + (it % NIN) * IN_DBL;
      mbar_wait(&inBar[it % NIN], (uint32_t)((it / NIN) & 1));
      ET_MARK(it, 0, lane == 0);
      if (lane < CELLS) {
        double x[12];
#pragma unroll
        for (int r = 0; r < 12; ++r)  // cells past the end: reference tet (never stored)
          x[r] = lane < nt ? in[lane * 12 + r] : ((r == 3 || r == 7 || r == 11) ? 1.0 : 0.0);
        const Geo geo = cell_geometry(x);
        double* cd = sCell + lane * CELLD;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) cd[a * 3 + bb] = geo.K[a][bb];
        cd[9] = lane < nt ? geo.adet : 0.0;
      }
      if (it >= 2) et_nbar_sync(BAR_EMPTY + b, THREADS);
      ET_MARK(it, 1, lane == 0);
      __syncwarp();
      // lane -> MMA row r = 3 cell + u (15 rows; row 15 zero), both GEMMs:
      // off-diagonal block u -> (c,d) = (0,1) (0,2) (1,2); diagonal u -> (u,u)
      if (lane < 16) {
        const int r = lane, cell = r / 3, u = r % 3;
        const bool live = r < 15 && cell < nt;
        const double* cd = sCell + (r < 15 ? cell : 0) * CELLD;
        double Kc[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) Kc[i] = cd[i];
        const double ad = live ? cd[9] : 0.0;
        const double* cf = in + CELLS * 12 + 4 + (r < 15 ? cell : 0) * NCOEF;
        const int oc = u == 2 ? 1 : 0, od = u == 0 ? 1 : 2;
        const int ln = 4 * (r & 7), v = r >> 3;
#pragma unroll
        for (int aa = 0; aa < 9; ++aa) {
          const int a = aa / 3, a2 = aa % 3;
          const double kk = Kc[a * 3 + 0] * Kc[a2 * 3 + 0] + Kc[a * 3 + 1] * Kc[a2 * 3 + 1] +
                            Kc[a * 3 + 2] * Kc[a2 * 3 + 2];
          // off-diagonal (oc, od) and diagonal (u, u)
          const double Po = Kc[a * 3 + oc] * Kc[a2 * 3 + od];
          const double Qo = Kc[a * 3 + od] * Kc[a2 * 3 + oc];
          const double Pd = Kc[a * 3 + u] * Kc[a2 * 3 + u];
          const double Qd = Pd + kk;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const double mu = ad * cf[m], lam = ad * cf[4 + m];
            const int kap = m * 9 + aa;
            const int idx = ((kap >> 2) * 32 + ln + (kap & 3)) * 2 + v;
            AF[idx] = lam * Po + mu * Qo;
            AF[KS * 64 + idx] = lam * Pd + mu * Qd;
          }
        }
      } else {
        // row 15: zero (both GEMMs)
        const int r = 15, ln = 4 * (r & 7), v = r >> 3;
        for (int kap = lane - 16; kap < KD; kap += 16) {
          const int idx = ((kap >> 2) * 32 + ln + (kap & 3)) * 2 + v;
          AF[idx] = 0.0;
          AF[KS * 64 + idx] = 0.0;
        }
      }
      __syncwarp();
      fence_proxy_async();
      load(it + NIN);  // this tile's input buffer is consumed
      ET_MARK(it, 2, lane == 0);
      et_nbar_arrive(BAR_FULL + b, THREADS);
    }
    return;
  }

  // ======================= compute warps: three n8 tiles each =======================
  const bool issuer = warp == 0 && lane == 0;
  double bt[TPW][KS];
  int tj[TPW], tk[TPW];   // this lane's output slot (columns 2t, 2t+1) per tile
  bool tsym[TPW];
#pragma unroll
  for (int x = 0; x < TPW; ++x) {
    const int n = TPW * warp + x;  // 0..12 full, 13..20 diagonal half
    tsym[x] = n >= NF;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bt[x][ks] = tab[(n * KS + ks) * 32 + lane];
    if (!tsym[x]) {
      const int p = 8 * n + 2 * t;
      tj[x] = p < NS * NS ? p / NS : -1;
      tk[x] = p % NS;
    } else {
      const int sidx = 8 * (n - NF) + 2 * t;
      tj[x] = c_et_sym[sidx][0];
      tk[x] = c_et_sym[sidx][1];
    }
  }
  // the MMA rows this lane holds: g and g + 8 -> (cell, block)
  int rcell[2], ru[2];
#pragma unroll
  for (int vh = 0; vh < 2; ++vh) {
    const int r = g + 8 * vh;
    rcell[vh] = r < 15 ? r / 3 : -1;
    ru[vh] = r % 3;
  }

  for (long it = 0; it < my_tiles; ++it) {
    const long c0 = (blockIdx.x + it * gridDim.x) * CELLS;
    const int nt = (int)min((long)CELLS, E - c0);
    const int b = (int)(it & 1);
    const double2* AF = reinterpret_cast<const double2*>(sAF + b * AF_DBL);
    et_nbar_sync(BAR_FULL + b, THREADS);
    ET_MARK(it, 3, tid == 0);
    double acc4[TPW][4];
#pragma unroll
    for (int x = 0; x < TPW; ++x)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc4[x][v] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double2 ao = AF[ks * 32 + lane];
      const double2 ad = AF[(KS + ks) * 32 + lane];
#pragma unroll
      for (int x = 0; x < TPW; ++x) {
        const double2 af = tsym[x] ? ad : ao;
        et_dmma(acc4[x], af.x, af.y, bt[x][ks]);
      }
    }
    if (it + 2 < my_tiles) et_nbar_arrive(BAR_EMPTY + b, THREADS);
    ET_MARK(it, 4, tid == 0);
    double* stg = sStg + b * STG_DBL;
    if (issuer) bulk_wait_read1();  // the store of tile it-2 has left this buffer
    ET_MARK(it, 5, tid == 0);
    et_nbar_sync(BAR_C, CTHREADS);
    ET_MARK(it, 6, tid == 0);
    // acc4[x][v] = C[row g + 8(v>>1)][col 2t + (v&1)]
#pragma unroll
    for (int x = 0; x < TPW; ++x) {
      const int j = tj[x], k = tk[x];
      if (j < 0) continue;
#pragma unroll
      for (int vh = 0; vh < 2; ++vh) {
        if (rcell[vh] < 0) continue;
        double* cp = stg + rcell[vh] * N * N;
        const double e0 = acc4[x][2 * vh], e1 = acc4[x][2 * vh + 1];
        if (!tsym[x]) {
          const int c = ru[vh] == 2 ? 1 : 0, d = ru[vh] == 0 ? 1 : 2;
          // direct (c, j) x (d, k..k+1); mirror (d, k..k+1) x (c, j)
          *reinterpret_cast<double2*>(cp + (c * NS + j) * N + d * NS + k) = make_double2(e0, e1);
          cp[(d * NS + k) * N + c * NS + j] = e0;
          cp[(d * NS + k + 1) * N + c * NS + j] = e1;
        } else {
          const int c = ru[vh];
          double* blk = cp + c * NS * N + c * NS;
          // each upper entry once, mirrored once; slot (j, j-1) is the lower
          // duplicate of (j-1, j) and is left to that slot's mirror
          if (k >= j) blk[j * N + k] = e0;
          if (k > j) blk[k * N + j] = e0;
          if (k + 1 >= j) blk[j * N + k + 1] = e1;
          if (k + 1 > j) blk[(k + 1) * N + j] = e1;
        }
      }
    }
    fence_proxy_async();
    et_nbar_sync(BAR_C, CTHREADS);
    ET_MARK(it, 7, tid == 0);
    if (issuer) {
      if (acc)
        bulk_s2g_add(A + c0 * N * N, stg, nt * N * N * 8);
      else
        bulk_s2g(A + c0 * N * N, stg, nt * N * N * 8);
      bulk_commit();
    }
  }
  if (issuer) bulk_wait0();
}

// ---------------------------------------------------------------------------
bool elas_tensor_supported(int ns, int nc) { return ns == et::NS && nc == 4; }

size_t elas_tensor_table_doubles() { return et::TF_DBL; }

void elas_tensor_tables(int nq, const double* W, const double* D, const double* P, double* out) {
  using namespace et;
  auto Dv = [&](int a, int q, int j) { return D[((size_t)a * nq + q) * NS + j]; };
  // T[kappa][j][k]
  std::vector<double> T((size_t)KD * NS * NS, 0.0);
  for (int m = 0; m < 4; ++m)
    for (int a = 0; a < 3; ++a)
      for (int a2 = 0; a2 < 3; ++a2)
        for (int j = 0; j < NS; ++j)
          for (int k = 0; k < NS; ++k) {
            double s = 0.0;
            for (int q = 0; q < nq; ++q) s += W[q] * P[q * 4 + m] * Dv(a, q, j) * Dv(a2, q, k);
            T[((size_t)(m * 9 + a * 3 + a2) * NS + j) * NS + k] = s;
          }
  signed char sym[64][2];
  et_sym_table(sym);
  // B fragments b = B[kappa = 4ks + t][col g]
  for (int f = 0; f < NF; ++f)
    for (int ks = 0; ks < KS; ++ks)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3, p = 8 * f + g;
        out[(f * KS + ks) * 32 + lane] =
            p < NS * NS ? T[((size_t)(4 * ks + t) * NS + p / NS) * NS + p % NS] : 0.0;
      }
  for (int u = 0; u < NSYM; ++u)
    for (int ks = 0; ks < KS; ++ks)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3, s = 8 * u + g;
        const int j = sym[s][0], k = sym[s][1];
        out[((NF + u) * KS + ks) * 32 + lane] =
            j >= 0 ? T[((size_t)(4 * ks + t) * NS + j) * NS + k] : 0.0;
      }
}

cudaError_t launch_elas_tensor(long E, const double* coords, const double* coef, const double* tab,
                               double* A, int acc, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  static const char once_key = 0;  // one per (kernel instantiation, device)
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(elas_tensor_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)et::SMEM);
    if (e != cudaSuccess) return e;
    signed char sym[64][2];
    et_sym_table(sym);
    e = cudaMemcpyToSymbol(c_et_sym, sym, sizeof sym);
    if (e != cudaSuccess) return e;
    return cudaSuccess;
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + et::CELLS - 1) / et::CELLS;
  const long maxc = (long)et::CTAS_PER_SM * num_sms();
  const int grid = (int)(ntiles < maxc ? ntiles : maxc);
  elas_tensor_kernel<<<grid, et::THREADS, et::SMEM, s>>>(E, coords, coef, tab, A, acc);
  return cudaGetLastError();
}

}  // namespace femgpu
