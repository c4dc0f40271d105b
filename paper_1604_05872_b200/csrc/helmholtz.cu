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
// P1: thread per cell, persistent CTAs, TMA bulk-copy input ring
// ============================================================================
#ifndef P1_TILE_CELLS
#define P1_TILE_CELLS 128
#endif
#ifndef P1_STAGES
#define P1_STAGES 2  // c1, 2000 launches from one CUDA graph (us per launch), tile x stages x
                     // CTAs/SM: 128x2x2 62.8; 64x2x3 66.1; 64x4x2 67.0; 128x3x2 73.4; 128x3x3 73.6
#endif
#ifndef P1_CTAS_PER_SM
#define P1_CTAS_PER_SM 2
#endif
constexpr int P1_TILE = P1_TILE_CELLS;  // cells per tile = threads per CTA
constexpr int P1_NBUF = P1_STAGES;      // input stages in flight per CTA
constexpr int P1_CTAS = P1_CTAS_PER_SM; // CTAs per SM
constexpr int P1_SO = 18;         // padded output staging stride: conflict-free 16B stores
constexpr int P1_IN = P1_TILE * 16;                       // doubles per input stage
constexpr size_t P1_SMEM = sizeof(double) * (P1_NBUF * P1_IN + P1_TILE * P1_SO) +
                           P1_NBUF * sizeof(uint64_t);

template <bool ACC>
__global__ void __launch_bounds__(P1_TILE, P1_CTAS)
    helm_p1_kernel(HelmP1Params prm, long E, const double* __restrict__ coords,
                   const double* __restrict__ coef, double* __restrict__ A,
                   const long* __restrict__ pos, double* __restrict__ vals) {
  extern __shared__ __align__(16) double smem[];
  double* sIn = smem;                               // [NBUF][coords 128x12 | f 128x4]
  double* so = smem + P1_NBUF * P1_IN;              // [128][18]
  uint64_t* full = reinterpret_cast<uint64_t*>(so + P1_TILE * P1_SO);
  const int tid = threadIdx.x;
  const long ntiles = (E + P1_TILE - 1) / P1_TILE;
  if ((long)blockIdx.x >= ntiles) return;
  if (tid == 0) {
    for (int b = 0; b < P1_NBUF; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long tile, int b) {  // both inputs of a tile: contiguous, 16B multiples
    const long e0 = tile * P1_TILE;
    const int nt = (int)min((long)P1_TILE, E - e0);
    double* dst = sIn + b * P1_IN;
    mbar_expect_tx(&full[b], nt * 128);
    bulk_g2s(dst, coords + e0 * 12, nt * 96, &full[b]);
    bulk_g2s(dst + P1_TILE * 12, coef + e0 * 4, nt * 32, &full[b]);
  };
  if (tid == 0)
    for (int b = 0; b < P1_NBUF; ++b) {
      const long tl = blockIdx.x + (long)b * gridDim.x;
      if (tl < ntiles) issue(tl, b);
    }
  long it = 0;
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = (int)(it % P1_NBUF);
    const long e0 = tile * P1_TILE;
    const int nt = (int)min((long)P1_TILE, E - e0);
    mbar_wait(&full[b], (uint32_t)((it / P1_NBUF) & 1));
    const double* sx = sIn + b * P1_IN;
    const double* sf = sx + P1_TILE * 12;
    if (tid < nt) {
      double x[12];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const double2 v = reinterpret_cast<const double2*>(sx + tid * 12)[i];
        x[2 * i] = v.x;
        x[2 * i + 1] = v.y;
      }
      const double2 f01 = reinterpret_cast<const double2*>(sf + tid * 4)[0];
      const double2 f23 = reinterpret_cast<const double2*>(sf + tid * 4)[1];
      const double f[4] = {f01.x, f01.y, f23.x, f23.y};
      const Geo geo = cell_geometry(x);
      double g[4][3];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int bb = 0; bb < 3; ++bb)
          g[j][bb] = geo.K[0][bb] * prm.Dr[j][0] + geo.K[1][bb] * prm.Dr[j][1] +
                     geo.K[2][bb] * prm.Dr[j][2];
      const double fbar = f[0] * prm.c[0] + f[1] * prm.c[1] + f[2] * prm.c[2] + f[3] * prm.c[3];
      double out[16];
      int p = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = j; k < 4; ++k, ++p) {
          const double st = g[j][0] * g[k][0] + g[j][1] * g[k][1] + g[j][2] * g[k][2];
          const double ms = f[0] * prm.M[0][p] + f[1] * prm.M[1][p] + f[2] * prm.M[2][p] +
                            f[3] * prm.M[3][p];
          const double v = geo.adet * (fbar * st + ms);
          out[j * 4 + k] = v;
          out[k * 4 + j] = v;
        }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<double2*>(&so[tid * P1_SO + 2 * i]) = make_double2(out[2 * i], out[2 * i + 1]);
    }
    __syncthreads();  // staging complete; input stage b fully consumed
    if (tid == 0) {
      const long nx = tile + (long)P1_NBUF * gridDim.x;
      if (nx < ntiles) issue(nx, b);
    }
    double2* gA = reinterpret_cast<double2*>(A + e0 * 16);
    double2 v[8];  // all 8 staged loads in flight before the streaming stores
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = u * P1_TILE + tid;
      if (i < nt * 8) v[u] = *reinterpret_cast<const double2*>(&so[(i / 8) * P1_SO + 2 * (i % 8)]);
    }
    __syncthreads();  // staging free for the next tile
    if (pos) {  // fused global assembly: vals[pos] += A_e (CSR positions, global.cu)
      const long* gp = pos + e0 * 16;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = u * P1_TILE + tid;
        if (i < nt * 8) {
          const longlong2 p = ldg_stream_idx(reinterpret_cast<const longlong2*>(gp) + i);
          atomicAdd(vals + p.x, v[u].x);
          atomicAdd(vals + p.y, v[u].y);
        }
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = u * P1_TILE + tid;
      if (i < nt * 8) {
        if (ACC) {
          const double2 o = gA[i];
          v[u].x += o.x;
          v[u].y += o.y;
        }
        stg_stream(gA + i, v[u]);
      }
    }
  }
}

cudaError_t launch_helm_p1(const HelmP1Params& prm, long E, const double* coords,
                           const double* coef, double* A, int acc, cudaStream_t s,
                           const long* pos, double* vals) {
  if (E <= 0) return cudaSuccess;
  static const char once_key = 0;  // one per (kernel instantiation, device)
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    for (auto fn : {helm_p1_kernel<false>, helm_p1_kernel<true>}) {
      cudaError_t e =
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P1_SMEM);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + P1_TILE - 1) / P1_TILE;
  const long maxc = (long)P1_CTAS * num_sms();
  const int grid = (int)(ntiles < maxc ? ntiles : maxc);
  if (acc)
    helm_p1_kernel<true><<<grid, P1_TILE, P1_SMEM, s>>>(prm, E, coords, coef, A, pos, vals);
  else
    helm_p1_kernel<false><<<grid, P1_TILE, P1_SMEM, s>>>(prm, E, coords, coef, A, pos, vals);
  return cudaGetLastError();
}

// ============================================================================
// Tensor schedule on the FP64 tensor cores -- warp-specialised, persistent
// ============================================================================
//   warps 0..7   MMA: C[32 cells x 8*NT] += g (smem) x S (TMA ring), then drop
//                the symmetric half (j<=k) into a 32-cell staging tile
//   warps 8..11  IO:  inputs -> per-cell factors g (fragment-native, double
//                buffered) for the NEXT tile; mirrored, coalesced copy-out
//   warp  12     TMA producer: S k-chunks into a 3-stage ring (bulk copies)
// so the tensor cores never wait for a prologue or an epilogue.
#ifndef HT_KPS
#define HT_KPS 2
#endif
#ifndef HT_NBUF
#define HT_NBUF 3
#endif
template <int NS, int NC>
struct HelmTensorShape {
  static constexpr int NP = NS * (NS + 1) / 2;          // symmetric half of A_e
  static constexpr int NT = ((NP + 7) / 8 + 1) / 2 * 2;  // n8 tiles (even)
  static constexpr int KR = 7 * NC;                     // alpha = (m, s)
  static constexpr int KPS = HT_KPS;                    // k8 steps per pipeline stage
  static constexpr int KS = ((KR + 8 * KPS - 1) / (8 * KPS)) * KPS;  // k8 steps (padded)
  static constexpr int NSTG = KS / KPS;                 // stages per tile
  static constexpr int NBUF = HT_NBUF;                  // TMA ring depth
  static constexpr int MT = 2;                          // m16 tiles per CTA tile
  static constexpr int CELLS = 16 * MT;                 // cells per tile
  static constexpr int MMA_WARPS = 8;
  static constexpr int IO_WARPS = 4;
  static constexpr int IO_THREADS = 32 * IO_WARPS;
  static constexpr int THREADS = 32 * (MMA_WARPS + IO_WARPS + 1);
  static constexpr int NTW = (NT + MMA_WARPS - 1) / MMA_WARPS;  // max n8 tiles per MMA warp
  static constexpr int STAGE_DBL = KPS * NT * 64;       // doubles per ring stage
  static constexpr int A_DBL = MT * KS * 128;           // fragment-native g tile
  static constexpr int IN_DBL = CELLS * (12 + NC);      // raw inputs of a tile
  static constexpr int SP = NP + 2;                     // staging row: symmetric half only
  static constexpr int STG_DBL = CELLS * SP;
  static constexpr int NBAR = 2 * NBUF + 4 + 2;
  static constexpr size_t SMEM =
      sizeof(double) * (size_t)(2 * A_DBL + NBUF * STAGE_DBL + IN_DBL + STG_DBL) +
      NBAR * sizeof(uint64_t) + NS * NS * sizeof(short);
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void io_barrier(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

template <int NS, int NC>
__global__ void __launch_bounds__(HelmTensorShape<NS, NC>::THREADS, 1)
    helm_tensor_kernel(long E, const double* __restrict__ coords, const double* __restrict__ coef,
                       const double* __restrict__ Sfrag, double* __restrict__ A, int acc) {
  using Sh = HelmTensorShape<NS, NC>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;                                  // [2][MT][KS][32][4]
  double* sB = sA + 2 * Sh::A_DBL;                    // [NBUF][KPS][NT][32][2]
  double* sIn = sB + Sh::NBUF * Sh::STAGE_DBL;        // [CELLS][12] | [CELLS][NC]
  double* stg = sIn + Sh::IN_DBL;                     // [CELLS][SP] (j<=k half)
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + Sh::STG_DBL);
  uint64_t* bFull = bar;                              // [NBUF]  TMA -> MMA
  uint64_t* bEmpty = bar + Sh::NBUF;                  // [NBUF]  MMA -> producer
  uint64_t* aFull = bar + 2 * Sh::NBUF;               // [2]     IO -> MMA
  uint64_t* aEmpty = aFull + 2;                       // [2]     MMA -> IO
  uint64_t* sFull = aFull + 4;                        //         MMA -> IO (staging written)
  uint64_t* sEmpty = aFull + 5;                       //         IO -> MMA (staging drained)
  short* sPidx = reinterpret_cast<short*>(bar + Sh::NBAR);  // (j,k) -> p(min, max)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  if ((long)blockIdx.x >= ntiles) return;
  const long my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  if (tid == 0) {
    for (int b = 0; b < Sh::NBUF; ++b) {
      mbar_init(&bFull[b], 1);
      mbar_init(&bEmpty[b], Sh::MMA_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&aFull[b], Sh::IO_THREADS);
      mbar_init(&aEmpty[b], Sh::MMA_WARPS);
    }
    mbar_init(sFull, Sh::MMA_WARPS);
    mbar_init(sEmpty, Sh::IO_THREADS);
    fence_mbar_init();
  }
  for (int jk = tid; jk < NS * NS; jk += Sh::THREADS) {
    const int j = jk / NS, k = jk % NS;
    const int lo = j < k ? j : k, hi = j < k ? k : j;
    sPidx[jk] = (short)(lo * NS - lo * (lo - 1) / 2 + (hi - lo));
  }
  __syncthreads();

  if (warp < Sh::MMA_WARPS) {
    // ======================= MMA warps =======================
    const int g = lane >> 2, t = lane & 3;
    int ntw = 0;
    for (int x = warp; x < Sh::NT; x += Sh::MMA_WARPS) ++ntw;
    int cb_buf = 0, cb_phase = 0;  // ring position of the next stage to consume
    for (long it = 0; it < my_tiles; ++it) {
      const int ab = (int)(it & 1);
      mbar_wait(&aFull[ab], (uint32_t)((it >> 1) & 1));
      const double* sAb = sA + ab * Sh::A_DBL;
      double c[Sh::MT][Sh::NTW][4];
#pragma unroll
      for (int mt = 0; mt < Sh::MT; ++mt)
#pragma unroll
        for (int i = 0; i < Sh::NTW; ++i) c[mt][i][0] = c[mt][i][1] = c[mt][i][2] = c[mt][i][3] = 0.0;
#pragma unroll 1
      for (int st = 0; st < Sh::NSTG; ++st) {
        const int b = cb_buf;
        mbar_wait(&bFull[b], (uint32_t)cb_phase);
        const double* Bst = sB + b * Sh::STAGE_DBL;
#pragma unroll
        for (int kk = 0; kk < Sh::KPS; ++kk) {
          const int ks = st * Sh::KPS + kk;
          double a[Sh::MT][4];
#pragma unroll
          for (int mt = 0; mt < Sh::MT; ++mt) {
            // [mt][ks][half][32 lanes][2]: each 16-byte load is lane-contiguous
            const double2* ap = reinterpret_cast<const double2*>(sAb) + (mt * Sh::KS + ks) * 64 + lane;
            const double2 a01 = ap[0], a23 = ap[32];
            a[mt][0] = a01.x;
            a[mt][1] = a01.y;
            a[mt][2] = a23.x;
            a[mt][3] = a23.y;
          }
#pragma unroll
          for (int i = 0; i < Sh::NTW; ++i) {
            if (i < ntw) {
              const int ntile = warp + i * Sh::MMA_WARPS;
              const double2 bv =
                  reinterpret_cast<const double2*>(Bst)[(kk * Sh::NT + ntile) * 32 + lane];
              const double bb[2] = {bv.x, bv.y};
#pragma unroll
              for (int mt = 0; mt < Sh::MT; ++mt) dmma16x8x8(c[mt][i], a[mt], bb);
            }
          }
        }
        if (++cb_buf == Sh::NBUF) {
          cb_buf = 0;
          cb_phase ^= 1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bEmpty[b]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&aEmpty[ab]);
      // epilogue: the j<=k half of the tile into staging (the IO warps mirror it)
      mbar_wait(sEmpty, (uint32_t)(it & 1));
#pragma unroll
      for (int mt = 0; mt < Sh::MT; ++mt)
#pragma unroll
        for (int i = 0; i < Sh::NTW; ++i) {
          if (i < ntw) {
            const int ntile = warp + i * Sh::MMA_WARPS;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int row = 16 * mt + g + 8 * (v >> 1);
              const int p = ntile * 8 + 2 * t + (v & 1);
              if (p < Sh::NP) stg[row * Sh::SP + p] = c[mt][i][v];
            }
          }
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(sFull);
    }
  } else if (warp < Sh::MMA_WARPS + Sh::IO_WARPS) {
    // ======================= IO warps =======================
    const int io = tid - 32 * Sh::MMA_WARPS;
    mbar_arrive(sEmpty);  // staging starts empty (completes phase 0)
    auto prologue = [&](long it) {
      const long tile = blockIdx.x + it * gridDim.x;
      const long c0 = tile * Sh::CELLS;
      const int nt = (int)min((long)Sh::CELLS, E - c0);
      const int ab = (int)(it & 1);
      if (it >= 2) mbar_wait(&aEmpty[ab], (uint32_t)(((it >> 1) - 1) & 1));
      for (int i = io; i < nt * 12; i += Sh::IO_THREADS) cp_async8(&sIn[i], coords + c0 * 12 + i);
      for (int i = io; i < nt * NC; i += Sh::IO_THREADS)
        cp_async8(&sIn[Sh::CELLS * 12 + i], coef + c0 * NC + i);
      asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
      io_barrier(Sh::IO_THREADS);
      double* sAb = sA + ab * Sh::A_DBL;
      constexpr int PARTS = Sh::IO_THREADS / Sh::CELLS;  // threads per cell
      constexpr int MPT = (NC + PARTS - 1) / PARTS;
      const int cell = io / PARTS, part = io % PARTS;
      if (cell < Sh::CELLS) {
        double Gs[7];
        double fv[MPT];
        if (cell < nt) {
          const Geo geo = cell_geometry(&sIn[cell * 12]);
          const double(*K)[3] = geo.K;
#pragma unroll
          for (int s = 0; s < 6; ++s) {
            const int a = s < 3 ? s : (s == 5 ? 1 : 0);
            const int b = s < 3 ? s : (s == 3 ? 1 : 2);
            Gs[s] = geo.adet * (K[a][0] * K[b][0] + K[a][1] * K[b][1] + K[a][2] * K[b][2]);
          }
          Gs[6] = geo.adet;
#pragma unroll
          for (int i = 0; i < MPT; ++i) {
            const int m = part + PARTS * i;
            fv[i] = m < NC ? sIn[Sh::CELLS * 12 + cell * NC + m] : 0.0;
          }
        } else {
#pragma unroll
          for (int s = 0; s < 7; ++s) Gs[s] = 0.0;
#pragma unroll
          for (int i = 0; i < MPT; ++i) fv[i] = 0.0;
        }
        const int cmt = cell >> 4, rr = cell & 15;
        const int gg = rr & 7, vrow = rr >> 3;
#pragma unroll
        for (int i = 0; i < MPT; ++i) {
          const int m = part + PARTS * i;
          if (m < NC) {
#pragma unroll
            for (int s = 0; s < 7; ++s) {
              const int alpha = m * 7 + s;
              const int ks = alpha >> 3, kk = alpha & 7;
              const int ln = gg * 4 + (kk & 3), v = vrow + 2 * (kk >> 2);
              sAb[(((cmt * Sh::KS + ks) * 2 + (v >> 1)) * 32 + ln) * 2 + (v & 1)] = fv[i] * Gs[s];
            }
          }
        }
        for (int alpha = Sh::KR + part; alpha < 8 * Sh::KS; alpha += PARTS) {  // zero K padding
          const int ks = alpha >> 3, kk = alpha & 7;
          const int ln = gg * 4 + (kk & 3), v = vrow + 2 * (kk >> 2);
          sAb[(((cmt * Sh::KS + ks) * 2 + (v >> 1)) * 32 + ln) * 2 + (v & 1)] = 0.0;
        }
      }
      io_barrier(Sh::IO_THREADS);  // sIn free for the next prologue
      mbar_arrive(&aFull[ab]);
    };
    prologue(0);
    for (long it = 0; it < my_tiles; ++it) {
      if (it + 1 < my_tiles) prologue(it + 1);
      const long c0 = (blockIdx.x + it * gridDim.x) * Sh::CELLS;
      {
        mbar_wait(sFull, (uint32_t)(it & 1));
        const long cb = c0;
        const int ncell = (int)min((long)Sh::CELLS, E - cb);
        constexpr int PER = NS * NS / 2;  // double2 per cell
        const int total = ncell * PER;
        double2* gA = reinterpret_cast<double2*>(A + cb * NS * NS);
        constexpr int U = 4;
        for (int base = 0; base < total; base += U * Sh::IO_THREADS) {
          double2 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = base + u * Sh::IO_THREADS + io;
            if (i < total) {  // mirror: A[j][k] = A[k][j] = staged p(min, max)
              const double* row = stg + (i / PER) * Sh::SP;
              const int jk = 2 * (i % PER);
              v[u] = make_double2(row[sPidx[jk]], row[sPidx[jk + 1]]);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = base + u * Sh::IO_THREADS + io;
            if (i < total) {
              if (acc) {
                const double2 o = gA[i];
                v[u].x += o.x;
                v[u].y += o.y;
              }
              stg_stream(gA + i, v[u]);
            }
          }
        }
        mbar_arrive(sEmpty);
      }
    }
  } else if (lane == 0) {
    // ======================= TMA producer =======================
    const long total_loads = my_tiles * Sh::NSTG;
    for (long i = 0; i < total_loads; ++i) {
      const int b = (int)(i % Sh::NBUF);
      if (i >= Sh::NBUF) mbar_wait(&bEmpty[b], (uint32_t)(((i / Sh::NBUF) - 1) & 1));
      const int chunk = (int)(i % Sh::NSTG);
      mbar_expect_tx(&bFull[b], Sh::STAGE_DBL * 8);
      bulk_g2s(sB + b * Sh::STAGE_DBL, Sfrag + (size_t)chunk * Sh::STAGE_DBL, Sh::STAGE_DBL * 8,
               &bFull[b]);
    }
  }
}

template <int NS, int NC>
static cudaError_t launch_tensor_t(long E, const double* coords, const double* coef,
                                   const double* Sfrag, double* A, int acc, cudaStream_t s) {
  using Sh = HelmTensorShape<NS, NC>;
  static const char once_key = 0;  // one per (kernel instantiation, device)
  const cudaError_t e0 = once_per_device(&once_key, [&]() -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(helm_tensor_kernel<NS, NC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM);
    if (e != cudaSuccess) return e;
    return cudaSuccess;
  });
  if (e0 != cudaSuccess) return e0;
  const long ntiles = (E + Sh::CELLS - 1) / Sh::CELLS;
  const long max_ctas = num_sms();  // persistent: one warp-specialised CTA per SM
  const int grid = (int)(ntiles < max_ctas ? ntiles : max_ctas);
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
  if (ns == 20 && nc == 20) return launch_tensor_t<20, 20>(E, coords, coef, Sfrag, A, acc, s);
  if (ns == 10 && nc == 10) return launch_tensor_t<10, 10>(E, coords, coef, Sfrag, A, acc, s);
  if (ns == 10 && nc == 4) return launch_tensor_t<10, 4>(E, coords, coef, Sfrag, A, acc, s);
  return cudaErrorInvalidValue;
}

}  // namespace femgpu
