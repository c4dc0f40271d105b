// helmholtz.cu -- weighted Helmholtz element kernels (BASELINE configs 1 and 2).
//
//   a(u,v) = int f (grad u . grad v + u v) dx,  f = sum_m f_m P_m.
//
// The reference reaches this form's element matrix through femopt's emitted
// loop nest (proj/src/emit_c.cpp:108-174).  For the G-factored encoding femopt
// pre-evaluates every monomial (1,442 and 160,322
// flops/cell) into A[e] += sum_alpha g_alpha(e) T_alpha (preeval.cpp:279-451,
// symbolic_reduce :190-277).  Both kernels here realise that TENSOR schedule,
// re-cut for the GPU:
//
//  * helm_p1_kernel (P1 basis, constant reference gradients): thread per cell,
//    A_jk = |det| ( fbar g_j.g_k + sum_m f_m M_m,jk ),  fbar = sum_m f_m c_m,
//    with c_m = sum_q W P_m and M_m,jk = sum_q W P_m B_j B_k pre-evaluated.
//    ~250 flops for 256 B of HBM traffic: HBM-bound.  Inputs and outputs are
//    staged through padded shared memory so every global access is a
//    coalesced 16-byte vector access.
//
//  * helm_tensor_kernel<NS,NC> (any degree): the contraction
//        A_e[p] = sum_alpha g_e[alpha] S[alpha][p],   p = (j<=k),
//        alpha = (m, s): g = f_m * Gsym_s,  Gsym = |det| (K K^T)_{00,11,22,01,02,12}, |det|
//    is a (cells x 7 NC) x (7 NC x NS(NS+1)/2) FP64 GEMM run on the tensor
//    cores (mma.sync m16n8k8 f64 -> DMMA) with the symmetric half only (A_e
//    and G are symmetric), mirrored in the epilogue.  S streams through a
//    3-stage TMA bulk-copy pipeline from L2; per-cell factors g are computed
//    in the prologue straight into fragment-native shared memory.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

// ============================================================================
// P1: thread per cell
// ============================================================================
constexpr int P1_TILE = 128;
constexpr int P1_SX = 14;  // padded smem strides (doubles): conflict-free 16B accesses
constexpr int P1_SF = 6;
constexpr int P1_SO = 18;

__global__ void __launch_bounds__(P1_TILE) helm_p1_kernel(HelmP1Params prm, long E,
                                                          const double* __restrict__ coords,
                                                          const double* __restrict__ coef,
                                                          double* __restrict__ A, int acc) {
  __shared__ __align__(16) double sx[P1_TILE * P1_SX];
  __shared__ __align__(16) double sf[P1_TILE * P1_SF];
  __shared__ __align__(16) double so[P1_TILE * P1_SO];
  const long e0 = (long)blockIdx.x * P1_TILE;
  const int nt = (int)min((long)P1_TILE, E - e0);
  const int tid = threadIdx.x;
  {
    const double2* gx = reinterpret_cast<const double2*>(coords + e0 * 12);
    for (int i = tid; i < nt * 6; i += P1_TILE) {
      double2 v = ldg_stream(gx + i);
      *reinterpret_cast<double2*>(&sx[(i / 6) * P1_SX + 2 * (i % 6)]) = v;
    }
    const double2* gf = reinterpret_cast<const double2*>(coef + e0 * 4);
    for (int i = tid; i < nt * 2; i += P1_TILE) {
      double2 v = ldg_stream(gf + i);
      *reinterpret_cast<double2*>(&sf[(i / 2) * P1_SF + 2 * (i % 2)]) = v;
    }
  }
  __syncthreads();
  if (tid < nt) {
    const Geo geo = cell_geometry(&sx[tid * P1_SX]);
    const double f[4] = {sf[tid * P1_SF + 0], sf[tid * P1_SF + 1], sf[tid * P1_SF + 2],
                         sf[tid * P1_SF + 3]};
    double g[4][3];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        g[j][b] = geo.K[0][b] * prm.Dr[j][0] + geo.K[1][b] * prm.Dr[j][1] +
                  geo.K[2][b] * prm.Dr[j][2];
    const double fbar = f[0] * prm.c[0] + f[1] * prm.c[1] + f[2] * prm.c[2] + f[3] * prm.c[3];
    double out[16];
    int p = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int k = j; k < 4; ++k, ++p) {
        double st = g[j][0] * g[k][0] + g[j][1] * g[k][1] + g[j][2] * g[k][2];
        double ms = f[0] * prm.M[0][p] + f[1] * prm.M[1][p] + f[2] * prm.M[2][p] +
                    f[3] * prm.M[3][p];
        double v = geo.adet * (fbar * st + ms);
        out[j * 4 + k] = v;
        out[k * 4 + j] = v;
      }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      *reinterpret_cast<double2*>(&so[tid * P1_SO + 2 * i]) = make_double2(out[2 * i], out[2 * i + 1]);
  }
  __syncthreads();
  double2* gA = reinterpret_cast<double2*>(A + e0 * 16);
  for (int i = tid; i < nt * 8; i += P1_TILE) {
    double2 v = *reinterpret_cast<const double2*>(&so[(i / 8) * P1_SO + 2 * (i % 8)]);
    if (acc) {
      double2 o = gA[i];
      v.x += o.x;
      v.y += o.y;
    }
    stg_stream(gA + i, v);
  }
}

cudaError_t launch_helm_p1(const HelmP1Params& prm, long E, const double* coords,
                           const double* coef, double* A, int acc, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  long grid = (E + P1_TILE - 1) / P1_TILE;
  helm_p1_kernel<<<(unsigned)grid, P1_TILE, 0, s>>>(prm, E, coords, coef, A, acc);
  return cudaGetLastError();
}

// ============================================================================
// Tensor schedule on the FP64 tensor cores
// ============================================================================
template <int NS, int NC>
struct HelmTensorShape {
  static constexpr int NP = NS * (NS + 1) / 2;          // symmetric half of A_e
  static constexpr int NT = ((NP + 15) / 16) * 2;       // n8 tiles, even (2 n-halves)
  static constexpr int NTW = NT / 2;                    // n8 tiles per warp
  static constexpr int KR = 7 * NC;                     // alpha = (m, s)
  static constexpr int KPS = 2;                         // k8 steps per pipeline stage
  static constexpr int KS = ((KR + 8 * KPS - 1) / (8 * KPS)) * KPS;  // k8 steps (padded)
  static constexpr int NSTG = KS / KPS;                 // stages per tile
  static constexpr int NBUF = 3;                        // pipeline depth
  static constexpr int MT = 4;                          // m16 tiles per CTA
  static constexpr int CELLS = 16 * MT;                 // cells per CTA tile
  static constexpr int THREADS = 256;                   // 8 warps = MT x 2 n-halves
  static constexpr int STAGE_DBL = KPS * NT * 64;       // doubles per B stage
  static constexpr int A_DBL = MT * KS * 128;           // fragment-native g tile
  static constexpr int IN_DBL = CELLS * (12 + NC);      // raw inputs of a tile
  static constexpr int STAGE_OUT_DBL = 16 * NS * NS;    // epilogue staging (aliases A)
  static_assert(STAGE_OUT_DBL <= A_DBL, "epilogue staging must fit in the A region");
  static constexpr size_t SMEM = sizeof(double) * (size_t)(A_DBL + NBUF * STAGE_DBL + IN_DBL) +
                                 NBUF * sizeof(uint64_t) + NP * sizeof(int);
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

template <int NS, int NC>
__global__ void __launch_bounds__(256, 1)
    helm_tensor_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                       const double* __restrict__ Sfrag, double* __restrict__ A, int acc) {
  using Sh = HelmTensorShape<NS, NC>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;                                  // [MT][KS][32][4]
  double* sB = sA + Sh::A_DBL;                        // [NBUF][KPS][NT][32][2]
  double* sIn = sB + Sh::NBUF * Sh::STAGE_DBL;        // [CELLS][12] then [CELLS][NC]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sIn + Sh::IN_DBL);
  int* sPair = reinterpret_cast<int*>(bar + Sh::NBUF);  // p -> (j*NS+k) | (k*NS+j) << 16

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mt = warp & 3, nh = warp >> 2;
  const int g = lane >> 2, t = lane & 3;
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  if ((long)blockIdx.x >= ntiles) return;

  if (tid == 0) {
    for (int b = 0; b < Sh::NBUF; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  for (int j = 0, p = 0; j < NS; ++j)
    for (int k = j; k < NS; ++k, ++p)
      if (p % Sh::THREADS == tid) sPair[p] = (j * NS + k) | ((k * NS + j) << 16);
  __syncthreads();
  // Stage loads this CTA will consume; never leave a bulk copy in flight at exit.
  const long my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const long total_loads = my_tiles * Sh::NSTG;
  // B pipeline: stage loads are numbered globally; load i carries k-chunk i % NSTG.
  long issued = 0;
  auto issue = [&](long i) {
    const int b = (int)(i % Sh::NBUF);
    const int chunk = (int)(i % Sh::NSTG);
    mbar_expect_tx(&bar[b], Sh::STAGE_DBL * 8);
    bulk_g2s(sB + b * Sh::STAGE_DBL, Sfrag + (size_t)chunk * Sh::STAGE_DBL, Sh::STAGE_DBL * 8,
             &bar[b]);
  };
  if (tid == 0)
    for (; issued < Sh::NBUF && issued < total_loads; ++issued) issue(issued);
  long consumed = 0;

  // raw inputs of a tile -> sIn (cp.async, 8-byte granularity: any alignment/tail)
  auto load_inputs = [&](long tile) {
    const long c0 = tile * Sh::CELLS;
    const int nt = (int)min((long)Sh::CELLS, E - c0);
    for (int i = tid; i < nt * 12; i += Sh::THREADS) cp_async8(&sIn[i], coords + c0 * 12 + i);
    for (int i = tid; i < nt * NC; i += Sh::THREADS)
      cp_async8(&sIn[Sh::CELLS * 12 + i], coef + c0 * NC + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  load_inputs(blockIdx.x);

  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long c0 = tile * Sh::CELLS;
    const int nt = (int)min((long)Sh::CELLS, E - c0);
    cp_async_wait_all();
    __syncthreads();
    // ---- prologue: g[cell][alpha] -> sA (fragment-native), 4 threads per cell
    {
      const int cell = tid >> 2, part = tid & 3;
      double Gs[7];
      double fv[(NC + 3) / 4];
      if (cell < nt) {
        const Geo geo = cell_geometry(&sIn[cell * 12]);
        const double(*K)[3] = geo.K;
        const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
#pragma unroll
        for (int s = 0; s < 6; ++s) {
          const int a = ab[s][0], b = ab[s][1];
          Gs[s] = geo.adet * (K[a][0] * K[b][0] + K[a][1] * K[b][1] + K[a][2] * K[b][2]);
        }
        Gs[6] = geo.adet;
#pragma unroll
        for (int i = 0; i < (NC + 3) / 4; ++i) {
          const int m = part + 4 * i;
          fv[i] = m < NC ? sIn[Sh::CELLS * 12 + cell * NC + m] : 0.0;
        }
      } else {
#pragma unroll
        for (int s = 0; s < 7; ++s) Gs[s] = 0.0;
#pragma unroll
        for (int i = 0; i < (NC + 3) / 4; ++i) fv[i] = 0.0;
      }
      const int cmt = cell >> 4, rr = cell & 15;
      const int gg = rr & 7, vrow = rr >> 3;
#pragma unroll
      for (int i = 0; i < (NC + 3) / 4; ++i) {
        const int m = part + 4 * i;
        if (m >= NC) break;
#pragma unroll
        for (int s = 0; s < 7; ++s) {
          const int alpha = m * 7 + s;
          const int ks = alpha >> 3, kk = alpha & 7;
          const int ln = gg * 4 + (kk & 3), v = vrow + 2 * (kk >> 2);
          sA[((cmt * Sh::KS + ks) * 32 + ln) * 4 + v] = fv[i] * Gs[s];
        }
      }
      // zero the K padding [KR, 8*KS)
      for (int alpha = Sh::KR + part; alpha < 8 * Sh::KS; alpha += 4) {
        const int ks = alpha >> 3, kk = alpha & 7;
        const int ln = gg * 4 + (kk & 3), v = vrow + 2 * (kk >> 2);
        sA[((cmt * Sh::KS + ks) * 32 + ln) * 4 + v] = 0.0;
      }
    }
    __syncthreads();
    // prefetch the next tile's raw inputs while the tensor cores run
    if (tile + gridDim.x < ntiles) load_inputs(tile + gridDim.x);

    // ---- main loop: C[16 x 8*NTW] per warp on the FP64 tensor cores
    double c[Sh::NTW][4];
#pragma unroll
    for (int i = 0; i < Sh::NTW; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int st = 0; st < Sh::NSTG; ++st) {
      const int b = (int)(consumed % Sh::NBUF);
      mbar_wait(&bar[b], (uint32_t)((consumed / Sh::NBUF) & 1));
      const double* Bst = sB + b * Sh::STAGE_DBL;
#pragma unroll
      for (int kk = 0; kk < Sh::KPS; ++kk) {
        const int ks = st * Sh::KPS + kk;
        double a[4];
        const double2* ap = reinterpret_cast<const double2*>(&sA[((mt * Sh::KS + ks) * 32 + lane) * 4]);
        double2 a01 = ap[0], a23 = ap[1];
        a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
        const double2* bp =
            reinterpret_cast<const double2*>(&Bst[((kk * Sh::NT + nh * Sh::NTW) * 32 + lane) * 2]);
#pragma unroll
        for (int i = 0; i < Sh::NTW; ++i) {
          double2 bv = bp[i * 32];
          double bb[2] = {bv.x, bv.y};
          dmma16x8x8(c[i], a, bb);
        }
      }
      ++consumed;
      __syncthreads();
      if (tid == 0 && issued < total_loads) issue(issued++);
    }

    // ---- epilogue: mirror the symmetric half into 16-cell staging, coalesced stores
    double* stg = sA;  // A region is dead until the next prologue
#pragma unroll 1
    for (int r = 0; r < Sh::MT; ++r) {
      if (mt == r) {
#pragma unroll
        for (int i = 0; i < Sh::NTW; ++i) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int row = g + 8 * (v >> 1);
            const int p = (nh * Sh::NTW + i) * 8 + 2 * t + (v & 1);
            if (p < Sh::NP) {
              const int jk = sPair[p];
              stg[row * NS * NS + (jk & 0xffff)] = c[i][v];
              stg[row * NS * NS + (jk >> 16)] = c[i][v];
            }
          }
        }
      }
      __syncthreads();
      const long cb = c0 + r * 16;
      const int ncell = (int)max(0L, min(16L, E - cb));
      double2* gA = reinterpret_cast<double2*>(A + cb * NS * NS);
      const double2* s2 = reinterpret_cast<const double2*>(stg);
      for (int i = tid; i < ncell * NS * NS / 2; i += Sh::THREADS) {
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

template <int NS, int NC>
static cudaError_t launch_tensor_t(long E, const double* coords, const double* coef,
                                   const double* Sfrag, double* A, int acc, cudaStream_t s,
                                   int max_ctas) {
  using Sh = HelmTensorShape<NS, NC>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(helm_tensor_kernel<NS, NC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  const int grid = (int)(ntiles < (long)max_ctas ? ntiles : (long)max_ctas);
  helm_tensor_kernel<NS, NC><<<grid, Sh::THREADS, Sh::SMEM, s>>>(E, coords, coef, Sfrag, A, acc);
  return cudaGetLastError();
}

bool helm_tensor_supported(int ns, int nc) {
  return (ns == 20 && nc == 20) || (ns == 10 && nc == 10) || (ns == 10 && nc == 4);
}

void helm_tensor_geometry(int ns, int nc, int* KS, int* NT, int* KR, int* NP) {
  auto fill = [&](auto sh) {
    using Sh = decltype(sh);
    *KS = Sh::KS;
    *NT = Sh::NT;
    *KR = Sh::KR;
    *NP = Sh::NP;
  };
  if (ns == 20 && nc == 20) fill(HelmTensorShape<20, 20>{});
  else if (ns == 10 && nc == 10) fill(HelmTensorShape<10, 10>{});
  else fill(HelmTensorShape<10, 4>{});
}

cudaError_t launch_helm_tensor(int ns, int nc, long E, const double* coords, const double* coef,
                               const double* Sfrag, double* A, int acc, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  const int ctas = kNumSMs;  // persistent: one CTA per SM
  if (ns == 20 && nc == 20) return launch_tensor_t<20, 20>(E, coords, coef, Sfrag, A, acc, s, ctas);
  if (ns == 10 && nc == 10) return launch_tensor_t<10, 10>(E, coords, coef, Sfrag, A, acc, s, ctas);
  if (ns == 10 && nc == 4) return launch_tensor_t<10, 4>(E, coords, coef, Sfrag, A, acc, s, ctas);
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
