// gemm_f64.cu -- C[M][N] += A[M][K] * B[K][N] in FP64 on the tensor cores (DMMA).
//
// The contraction step of femopt's pre-evaluated (tensor) plans run through the
// generic IR backend (ir_backend.cpp, strategy "gemm"): a plan's innermost nest
//   A[e][j][k] += sum_t T_t[j][k] * p_t(e)
// (the reference tensors T_t of preeval.cpp:279-451 against per-cell products p_t
// of the element preheader) is the GEMM  C = P * T  with M = cells, K = terms,
// N = j*k entries; the generated preheader kernel writes P, this kernel contracts.
//
// Tiling: CTA 64 x 64 (4 warps, 2 x 2, warp tile 32 x 32 = 2 m16 x 4 n8 DMMA
// accumulators), K in chunks of 16 staged by cp.async into double-buffered shared
// tiles with padded strides (A rows 20 doubles, B rows 72: every fragment load of
// a warp touches each bank pair at most twice, the 2-wavefront minimum of an
// LDS.64).  A is [M][lda] with lda a multiple of 16 and zero columns past K, or
// transposed [Kpad][lda] (zero rows past K); B is [Kpad][ldb] zero-padded to the
// CTA tiles.  Rows of C past M and columns past N
// are not touched.
#include "common.cuh"
#include "femgpu_internal.h"

namespace femgpu {

namespace gm {
constexpr int BM = 64, BN = 64, BK = 16;
constexpr int SA = 20;  // A tile row stride (doubles)
constexpr int SB = 72;  // B tile row stride
constexpr int A_DBL = BM * SA, B_DBL = BK * SB;
}  // namespace gm

__device__ __forceinline__ void gm_dmma(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

__device__ __forceinline__ void gm_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

template <bool AT>
__global__ void __launch_bounds__(128) gemm_f64_acc_kernel(long M, int N, int K, int lda,
                                                           const double* __restrict__ A,
                                                           const double* __restrict__ B, int ldb,
                                                           double* __restrict__ C) {
  using namespace gm;
  // AT: A stored transposed, [K][lda] (column m of row k at A[k*lda + m]; the
  // producer of A writes it coalesced); the A tile is then staged [BK][BM] with
  // the B tile's padded stride
  __shared__ __align__(16) double sA[2][AT ? BK * SB : A_DBL];
  __shared__ __align__(16) double sB[2][B_DBL];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 1, wn = warp & 1;  // warp tile (32 rows, 32 cols)
  const long m0 = (long)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int nk = (K + BK - 1) / BK;

  auto stage = [&](int kc, int buf) {
    // A: 64 rows x 16 doubles = 512 16-byte chunks; B: 16 rows x 64 doubles = 512
    if (AT) {
      for (int i = tid; i < BK * BM / 2; i += 128) {
        const int r = i / (BM / 2), c2 = i % (BM / 2);
        double* dst = &sA[buf][r * SB + 2 * c2];
        const long col = m0 + 2 * c2;
        if (col + 1 < M)
          gm_cp16(dst, A + (long)(kc * BK + r) * lda + col);
        else
          *reinterpret_cast<double2*>(dst) =
              make_double2(col < M ? A[(long)(kc * BK + r) * lda + col] : 0.0, 0.0);
      }
    } else {
      for (int i = tid; i < BM * BK / 2; i += 128) {
        const int r = i / (BK / 2), c2 = i % (BK / 2);
        double* dst = &sA[buf][r * SA + 2 * c2];
        const long row = m0 + r;
        if (row < M)
          gm_cp16(dst, A + row * lda + kc * BK + 2 * c2);
        else
          *reinterpret_cast<double2*>(dst) = make_double2(0.0, 0.0);
      }
    }
    for (int i = tid; i < BK * BN / 2; i += 128) {
      const int r = i / (BN / 2), c2 = i % (BN / 2);
      gm_cp16(&sB[buf][r * SB + 2 * c2], B + (long)(kc * BK + r) * ldb + n0 + 2 * c2);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

  stage(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) {
      stage(kc + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const double* a = sA[buf] + (AT ? wm * 32 : (wm * 32) * SA);
    const double* b = sB[buf] + wn * 32;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double af[2][2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (AT) {
          af[i][0] = a[(4 * k4 + t) * SB + 16 * i + g];
          af[i][1] = a[(4 * k4 + t) * SB + 16 * i + g + 8];
        } else {
          af[i][0] = a[(16 * i + g) * SA + 4 * k4 + t];
          af[i][1] = a[(16 * i + g + 8) * SA + 4 * k4 + t];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b[(4 * k4 + t) * SB + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) gm_dmma(acc[i][j], af[i][0], af[i][1], bf[j]);
    }
    __syncthreads();  // this buffer is restaged two chunks on
  }
  // epilogue: C += acc (fragment c[v] = C[row g + 8(v>>1)][col 2t + (v&1)])
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int vh = 0; vh < 2; ++vh) {
      const long row = m0 + wm * 32 + 16 * i + g + 8 * vh;
      if (row >= M) continue;
      double* crow = C + row * (long)N;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = n0 + wn * 32 + 8 * j + 2 * t;
        if (col + 1 < N && (N & 1) == 0) {
          double2 o = *reinterpret_cast<const double2*>(crow + col);
          o.x += acc[i][j][2 * vh];
          o.y += acc[i][j][2 * vh + 1];
          *reinterpret_cast<double2*>(crow + col) = o;
        } else {
          if (col < N) crow[col] += acc[i][j][2 * vh];
          if (col + 1 < N) crow[col + 1] += acc[i][j][2 * vh + 1];
        }
      }
    }
}

int gemm_f64_tile_n() { return gm::BN; }
int gemm_f64_tile_k() { return gm::BK; }

cudaError_t launch_gemm_f64_acc(long M, int N, int K, int lda, const double* A, const double* B,
                                int ldb, double* C, cudaStream_t s, bool a_transposed) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (lda % 2 || ldb % gm::BN) return cudaErrorInvalidValue;
  if (!a_transposed && lda < (K + gm::BK - 1) / gm::BK * gm::BK) return cudaErrorInvalidValue;
  if (a_transposed && lda < M) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)((M + gm::BM - 1) / gm::BM), (unsigned)((N + gm::BN - 1) / gm::BN));
  if (a_transposed)
    gemm_f64_acc_kernel<true><<<grid, 128, 0, s>>>(M, N, K, lda, A, B, ldb, C);
  else
    gemm_f64_acc_kernel<false><<<grid, 128, 0, s>>>(M, N, K, lda, A, B, ldb, C);
  return cudaGetLastError();
}

}  // namespace femgpu
