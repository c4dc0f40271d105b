// femgpu_internal.h -- declarations shared by the host C ABI and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include <functional>
#include <string>

namespace femgpu {

// The thread-local message femgpu_last_error() returns (capi.cu).
void set_last_error(const std::string& message);

// Runs init() once per (key, current device) -- kernel attributes and __constant__
// tables live in each device's context -- under a process-wide lock, so concurrent
// first launches from several host threads never race a launch past the setup.
// Only a successful init is remembered.
cudaError_t once_per_device(const void* key, const std::function<cudaError_t()>& init);

// Pre-evaluated P1 Helmholtz tables (kernel parameters: constant bank).
struct HelmP1Params {
  double c[4];      // c_m = sum_q W_q P_m(q)
  double M[4][10];  // M_m,(j<=k) = sum_q W_q P_m(q) B_j(q) B_k(q)
  double Dr[4][3];  // constant reference gradients, Dr[j][a] = D[a][*][j]
};

// pos/vals non-null: fused global assembly (vals[pos] += A_e) instead of writing A
cudaError_t launch_helm_p1(const HelmP1Params& prm, long E, const double* coords,
                           const double* coef, double* A, int acc, cudaStream_t s,
                           const long* pos = nullptr, double* vals = nullptr);

bool helm_tensor_supported(int ns, int nc);
void helm_tensor_geometry(int ns, int nc, int* KS, int* NT, int* KR, int* NP);
cudaError_t launch_helm_tensor(int ns, int nc, long E, const double* coords, const double* coef,
                               const double* Sfrag, double* A, int acc, cudaStream_t s);

// Helmholtz in the quadrature schedule (helm_quad.cu); tab = [W | B | D | P].
bool helm_quad_supported(int ns, int nc);
cudaError_t launch_helm_quad(int ns, int nq, int nc, long E, const double* coords,
                             const double* coef, const double* tab, double* A, int acc,
                             cudaStream_t s);

// Vector forms on CUDA cores: per-(j<=k) pair accumulation over quadrature
// points (elasticity, St Venant-Kirchhoff).  tab = [W(Q) | D(3,Q,ns) | P(Q,4)].
struct PairParams {
  int kind;  // FEMGPU_ELASTICITY or FEMGPU_HYPERELASTICITY
  int nq;
};
bool pair_supported(int kind, int nq, int ns);
cudaError_t launch_pair(int kind, int nq, int ns, long E, const double* coords,
                        const double* coef, const double* tab, const double* htab, double* A,
                        int acc, cudaStream_t s);

// St Venant-Kirchhoff on the FP64 tensor cores (see svk_mma.cu): per cell two
// symmetric rank-1-per-point products and one 6 x 55 product over the quadrature
// points.  tab = [W(Q) | D(3,Q,ns) | P(Q,4)] as for launch_pair.
bool svk_mma_supported(int nq, int ns);
cudaError_t launch_svk_mma(int nq, int ns, long E, const double* coords, const double* coef,
                           const double* tab, double* A, int acc, cudaStream_t s);

// Burgers Jacobian in the quadrature schedule (see burgers_quad.cu).
// tab = [W(Q) | B(Q,ns) | D(3,Q,ns)].
bool burgers_quad_supported(int nq, int ns);
cudaError_t launch_burgers_quad(int nq, int ns, long E, const double* coords, const double* coef,
                                const double* tab, double nu, double dt, double* A, int acc,
                                cudaStream_t s);

// Linear elasticity tensor schedule (see elasticity.cu).
bool elas_tensor_supported(int ns, int nc);
size_t elas_tensor_table_doubles();
void elas_tensor_tables(int nq, const double* W, const double* D, const double* P, double* out);
cudaError_t launch_elas_tensor(long E, const double* coords, const double* coef, const double* tab,
                               double* A, int acc, cudaStream_t s);

// C[M][N] += A[M][K] * B[K][N] on DMMA (gemm_f64.cu): A [M][lda] (lda a multiple of 16,
// zero columns past K) or, a_transposed, [ceil16(K)][lda >= M] (zero rows past K);
// B zero-padded to [ceil16(K)][ldb], ldb a multiple of 64.
int gemm_f64_tile_n();
int gemm_f64_tile_k();
cudaError_t launch_gemm_f64_acc(long M, int N, int K, int lda, const double* A, const double* B,
                                int ldb, double* C, cudaStream_t s, bool a_transposed = false);

// Gather / symbolic / numeric global assembly (see global.cu).
cudaError_t launch_gather(long E, int ncoef, const double* V, const int* cells, const double* coef,
                          const int* coef_idx, double* coords, double* coeffs, cudaStream_t s);
cudaError_t launch_csr_positions(long E, int n, const int* dof, const long* row_ptr,
                                 const int* col_idx, long* pos, int* missing, cudaStream_t s);
cudaError_t launch_scatter_add(long total, const double* A, const long* pos, double* vals,
                               cudaStream_t s);
cudaError_t launch_csr_row_offsets(long E, int n, const int* dof, const long* row_ptr,
                                   const long* pos, uint16_t* loc, int* bad, cudaStream_t s);
cudaError_t launch_csr_gather_rows(long nrows, int n, int maxlen, const long* row_ptr,
                                   const long* inc_ptr, const int* inc, const uint16_t* loc,
                                   const double* A, int acc, double* vals, cudaStream_t s);

// Burgers tensor schedule (see burgers.cu).
bool burgers_supported(int nq, int ns);

// element vectors (vector.cu)
bool vector_supported(int kind, int ns, int nc);
int vector_table_qpad(int nq);  // Burgers residual: quadrature rows padded to its chunk
cudaError_t launch_vector(int kind, int nq, int ns, int nc, long E, const double* coords,
                          const double* coef, const double* tab, const double* consts, double* out,
                          int acc, cudaStream_t s);
size_t burgers_table_doubles();
// Returns the derivative-space rank used by GEMM-1, or -1 if unsupported.
int burgers_tables(int nq, const double* W, const double* B, const double* D, double* out);
cudaError_t launch_burgers(int ns, long E, const double* coords, const double* coef,
                           const double* tab, double nu, double dt, double* A, int acc,
                           cudaStream_t s);

}  // namespace femgpu
