/* femgpu -- B200-native finite element local assembly (sm_100a, FP64).
 *
 * Drop-in replacement for the per-element kernels the reference (femopt,
 * arXiv 1604.05872) emits as C.  Library conventions mirror libfemopt
 * (/root/reference/proj/include/femopt.h:1-76):
 *   - opaque handle (femopt_kernel, femopt.h:18)  ->  femgpu_form;
 *   - every function returns 0 on success or an error code, femopt's codes
 *     1-11 keep their meaning (femopt.h:20-33) and 12-14 add device errors;
 *   - the message of the most recent failure on the calling thread is
 *     femgpu_last_error() (femopt_last_error, femopt.h:72-74;
 *     thread_local in capi.cpp:13);
 *   - no C++ exception ever crosses this ABI (capi.cpp:33-46, `guarded`).
 * Handles are reentrant: distinct forms may be used concurrently, one form may
 * be used from several threads on distinct streams.
 *
 * Data layout (all FP64, cell-major, row-major inside a cell):
 *   coords [E][4][3]   vertex coordinates of each tetrahedron
 *   coeffs [E][ncoef]  coefficient dofs, per form (see femgpu_form_kind)
 *   A      [E][n][n]   element matrix (component-blocked for vector forms)
 */
#ifndef FEMGPU_H
#define FEMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct femgpu_form femgpu_form;

typedef enum femgpu_error {
  FEMGPU_OK = 0,
  FEMGPU_ERR_PARSE = 1,              /* femopt.h:22 (unused here)            */
  FEMGPU_ERR_UNKNOWN_LOOP = 2,       /* femopt.h:23 (unused here)            */
  FEMGPU_ERR_NOT_FEM_NEST = 3,       /* femopt.h:24: unsupported form shape  */
  FEMGPU_ERR_NON_DISTRIBUTABLE = 4,  /* femopt.h:25 (unused here)            */
  FEMGPU_ERR_NON_SEPARABLE = 5,      /* femopt.h:26 (unused here)            */
  FEMGPU_ERR_NOT_NORMAL_FORM = 6,    /* femopt.h:27 (unused here)            */
  FEMGPU_ERR_TOO_MANY_MONOMIALS = 7, /* femopt.h:28 (unused here)            */
  FEMGPU_ERR_INCONSISTENT_LAYOUT = 8,/* femopt.h:29: table shapes disagree   */
  FEMGPU_ERR_INVALID_ARG = 9,        /* femopt.h:30                          */
  FEMGPU_ERR_IO = 10,                /* femopt.h:31 (unused here)            */
  FEMGPU_ERR_INTERNAL = 11,          /* femopt.h:32                          */
  FEMGPU_ERR_CUDA = 12,              /* a CUDA runtime call failed           */
  FEMGPU_ERR_NO_DEVICE = 13,         /* no sm_100 device / kernel image      */
  FEMGPU_ERR_UNSUPPORTED = 14        /* valid form, no kernel for its size   */
} femgpu_error;

/* Forms (BASELINE.json configs).  `ncoef` is the per-cell coefficient width.
 *   HELMHOLTZ        a(u,v) = int f (grad u . grad v + u v)
 *                    scalar P_k (k = degree), f in P_{coef_degree}:
 *                    coeffs = f dofs [nc]
 *   ELASTICITY       a(u,v) = int 2 mu eps(u):eps(v) + lam div u div v
 *                    vector P_k, mu, lam in P1: coeffs = [mu(4), lam(4)]
 *   HYPERELASTICITY  St Venant-Kirchhoff tangent at displacement w:
 *                    int (grad du S + F dS[du]) : grad v,  F = I + grad w
 *                    coeffs = [w (3 x ns, component-blocked), mu(4), lam(4)]
 *   BURGERS          int du.v/dt + (du.grad)u.v + (u.grad)du.v + nu grad du:grad v
 *                    coeffs = u (3 x ns, component-blocked); consts = {nu, dt}
 */
typedef enum femgpu_form_kind {
  FEMGPU_HELMHOLTZ = 1,
  FEMGPU_ELASTICITY = 2,
  FEMGPU_HYPERELASTICITY = 3,
  FEMGPU_BURGERS = 4
} femgpu_form_kind;

/* Kernel schedules (the paper's two strategies, §3.2-3.3):
 *   TENSOR      pre-evaluated reference tensors contracted with per-cell
 *               geometry/coefficient factors (preeval.cpp:279-451)
 *   QUADRATURE  per-quadrature-point sharing-eliminated accumulation
 *               (sharing.cpp:409-607)
 *   QUADRATURE_MMA  the same per-point operands, with the sum over points
 *               run as dense FP64 tensor-core products per cell (St Venant-
 *               Kirchhoff: svk_mma.cu) instead of per-pair FMA streams
 * AUTO ranks every kernel this library has for the form by predicted time --
 * the roofline time max(flops / FP64 peak, bytes / HBM bandwidth) of the
 * kernel's own flop and byte counts on the current device, divided by the
 * fraction of that roofline the kernel was measured to reach on B200 -- and
 * takes the fastest, the GPU counterpart of femopt's theta_pre / theta_se plan
 * choice (proj/src/cost.cpp:61-116, driver.cpp:47-106).  TENSOR / QUADRATURE
 * take the best kernel of that schedule.  femgpu_form_schedules() lists the
 * ranking. */
typedef enum femgpu_schedule {
  FEMGPU_SCHED_AUTO = 0,
  FEMGPU_SCHED_TENSOR = 1,
  FEMGPU_SCHED_QUADRATURE = 2,
  FEMGPU_SCHED_QUADRATURE_MMA = 3
} femgpu_schedule;

/* Reference tables of a form: exactly the input tables femopt's IR carries
 * (paper_1604_05872_b200/ir.py), on the reference tetrahedron
 * (0,0,0),(1,0,0),(0,1,0),(0,0,1).  Host pointers; copied at create time. */
typedef struct femgpu_form_desc {
  int kind;             /* femgpu_form_kind */
  int nq;               /* quadrature points Q */
  int ns;               /* scalar basis functions per component */
  int nc;               /* coefficient basis functions (cols of P) */
  const double* W;      /* [Q] weights */
  const double* B;      /* [Q][ns] basis values */
  const double* D;      /* [3][Q][ns] reference gradients d/dX_a */
  const double* P;      /* [Q][nc] coefficient basis values */
  double consts[4];     /* BURGERS: {nu, dt}; others ignored */
  int schedule;         /* femgpu_schedule */
} femgpu_form_desc;

typedef struct femgpu_form_info {
  int n;                      /* element matrix is n x n */
  int ncoef;                  /* coefficient dofs per cell */
  int schedule;               /* schedule in use */
  double flops_per_cell;      /* FP64 flops the chosen kernels execute per cell */
  double bytes_per_cell;      /* compulsory HBM bytes: 8*(12 + ncoef + n*n) */
  int kernels_per_launch;     /* device kernels one femgpu_assemble launches */
  char kernel_name[64];       /* dominant kernel's name */
} femgpu_form_info;

/* One kernel the library could run for a form, with its cost model. */
typedef struct femgpu_schedule_info {
  char kernel_name[64];
  int schedule;                  /* FEMGPU_SCHED_TENSOR, _QUADRATURE or _QUADRATURE_MMA */
  int pipe;                      /* FP64 pipe: 0 = DFMA (CUDA cores), 1 = DMMA (tensor) */
  double flops_per_cell;         /* FP64 flops the kernel executes per cell */
  double bytes_per_cell;         /* compulsory HBM bytes per cell */
  double peak_flops;             /* the pipe's FP64 peak on the current device, flop/s */
  double peak_bytes;             /* HBM bandwidth of the current device, B/s */
  double efficiency;             /* measured fraction of the roofline (B200, profiles/) */
  double predicted_ns_per_cell;  /* max(flops/peak_flops, bytes/peak_bytes)/efficiency */
  int chosen;                    /* 1 for the kernel femgpu_form_create would pick */
} femgpu_schedule_info;

/* The kernels available for a form descriptor, ranked by predicted time
 * (fastest first; the one desc->schedule selects has chosen = 1).  Writes at
 * most cap entries; *count = number available.  Needs a current CUDA device
 * (its attributes give the peaks); uploads nothing. */
int femgpu_form_schedules(const femgpu_form_desc* desc, femgpu_schedule_info* out, int cap,
                          int* count);

/* Creates a form on the current CUDA device: validates the tables, computes
 * the schedule's pre-evaluated reference tensors on the host in FP64
 * (ascending-quadrature-point left folds, as preeval.cpp:269-274), and uploads
 * them.  *out must be released with femgpu_form_free(). */
int femgpu_form_create(const femgpu_form_desc* desc, femgpu_form** out);
void femgpu_form_free(femgpu_form* f);
int femgpu_form_get_info(const femgpu_form* f, femgpu_form_info* info);

/* Element matrices of cells [0, ncells) -- the hot path.  Device pointers
 * (cell-major layout above), stream = cudaStream_t (NULL = legacy default).
 * accumulate = 0 overwrites A; nonzero adds into it (the emitted-C `+=`
 * contract, emit_c.cpp:129).  Asynchronous: returns after enqueueing.  The
 * current device must be the form's (FEMGPU_ERR_INVALID_ARG otherwise).  Safe
 * to call from several host threads at once, including their first calls. */
int femgpu_assemble(const femgpu_form* f, long ncells, const double* coords,
                    const double* coeffs, double* A, int accumulate, void* stream);

/* Element VECTORS of the form's family (arity-1 nests, kernel.cpp:369-390; the
 * IR paper_1604_05872_b200/ir.py builds with build_vector), same tables, inputs
 * and conventions as femgpu_assemble, output b [E][n]:
 *   HELMHOLTZ        load vector        b_j     = int f phi_j
 *   HYPERELASTICITY  internal work      r_(c,j) = int (F S) : grad(phi_j e_c)
 *   BURGERS          residual           r_(c,j) = int (u_c/dt + (u.grad)u_c) phi_j
 *                                                 + nu grad u_c . grad phi_j
 * FEMGPU_ERR_UNSUPPORTED for ELASTICITY and for sizes without a kernel. */
int femgpu_assemble_vector(const femgpu_form* f, long ncells, const double* coords,
                           const double* coeffs, double* b, int accumulate, void* stream);

/* Same, from and to HOST memory: copies in, assembles and copies out in a
 * chunked multi-stream pipeline (the end-to-end path).  Synchronous.
 * Pinned host buffers give full PCIe bandwidth; pageable ones work too. */
int femgpu_assemble_host(const femgpu_form* f, long ncells, const double* coords,
                         const double* coeffs, double* A, int accumulate);

/* The emitted-C element-kernel interface (emit_c.cpp:127-141) through the
 * reference harness's uniform entry point (test_backend.cpp:62-73):
 *   o = outputs in name order, t = input tables in name order, c = constants,
 * with femopt's IR naming for this form (paper_1604_05872_b200/ir.py) and
 * HOST pointers.  Per-cell tables are the SoA e-tables (x{v}{c}[e], dofs);
 * reference tables (W, B, D*, P*, Dv*, Du*, Dw*) must equal, bit for bit, the
 * ones the form was created with (its kernels use device copies of those):
 * FEMGPU_ERR_INCONSISTENT_LAYOUT names the first table that differs.  Burgers
 * constants (dt, nu) must equal the form's likewise.  Outputs are accumulated
 * with `+=` like emitted C.
 * `ncells` replaces the literal E of the emitted code. */
int femgpu_kernel_argv(const femgpu_form* f, long ncells, double* const* o,
                       const double* const* t, const double* c);

/* Number and names of the arguments femgpu_kernel_argv expects, in order
 * (group: 0 = output, 1 = table, 2 = constant). */
int femgpu_kernel_argc(const femgpu_form* f, int group, int* count);
int femgpu_kernel_argname(const femgpu_form* f, int group, int index, char* buf, size_t len);

/* ---------------------------------------------------------------------------
 * Either side of the path (the reference reads
 * pre-gathered per-cell tables, proj/tests/kernels.hpp:186-188, and stops at
 * the element matrix).  All pointers are device pointers.
 * ------------------------------------------------------------------------- */

/* Gather the per-cell inputs of femgpu_assemble from global vectors:
 * coords[e][v][c] = V[cells[e][v]][c]  (cells: [ncells][4] vertex ids),
 * coeffs[e][s]    = coef[coef_idx[e][s]] (coef_idx: [ncells][ncoef]). */
int femgpu_gather(long ncells, int ncoef, const double* V, const int* cells, const double* coef,
                  const int* coef_idx, double* coords, double* coeffs, void* stream);

/* Symbolic assembly: pos[e][j][k] = position of column dof_map[e][k] in row
 * dof_map[e][j] of the CSR pattern (row_ptr [nrows+1], col_idx sorted per row).
 * Synchronizes the stream; FEMGPU_ERR_INCONSISTENT_LAYOUT if any entry of an
 * element matrix is outside the pattern. */
int femgpu_csr_positions(long ncells, int n, const int* dof_map, const long* row_ptr,
                         const int* col_idx, long* pos, void* stream);

/* Numeric assembly: vals[pos[i]] += A[i] for i < nentries (FP64 atomics;
 * A = the element matrices [ncells][n][n] of femgpu_assemble). */
int femgpu_scatter_add(long nentries, const double* A, const long* pos, double* vals,
                       void* stream);

/* Symbolic, once per mesh, for femgpu_csr_gather_rows: loc[e][j][k] =
 * pos[e][j][k] - row_ptr[dof_map[e][j]], the entry's offset inside its CSR row
 * (rows of at most 65536 entries).  Synchronizes the stream;
 * FEMGPU_ERR_INCONSISTENT_LAYOUT if an entry lies outside its row. */
int femgpu_csr_row_offsets(long ncells, int n, const int* dof_map, const long* row_ptr,
                           const long* pos, uint16_t* loc, void* stream);

/* Numeric assembly without atomics: one warp per CSR row r sums the element-matrix
 * rows incident to it -- inc[inc_ptr[r] .. inc_ptr[r+1]) holds the element-row ids
 * e*n + j with dof_map[e][j] == r -- in that order (bit-reproducible), then
 * writes the row once: vals (=, or += with accumulate).  n <= 64; max_row_len =
 * the longest CSR row. */
int femgpu_csr_gather_rows(long nrows, int n, const long* row_ptr, const long* inc_ptr,
                           const int* inc, const uint16_t* loc, int max_row_len,
                           const double* A, double* vals, int accumulate, void* stream);

/* ---------------------------------------------------------------------------
 * Any femopt kernel: the GPU counterpart of femopt's
 * emit_c backend (proj/src/emit_c.cpp:108-174).  femgpu_ir_create takes the
 * kernel IR JSON (proj/README.md:68-100, raw or as femopt_kernel_to_json writes
 * it), generates CUDA for it and compiles it with NVRTC for sm_100a.  Argument
 * groups and order are emit_c's: outputs, input tables, constants, each sorted
 * by name (emit_c.cpp:137-140); outputs are accumulated with +=.  The thread
 * and warp mappings are bit-identical to femopt's emitted C compiled with
 * -ffp-contract=off.  The GEMM mapping applies to femopt's pre-evaluated
 * (tensor) plans -- an element body of scalar statements followed by one nest
 * OUT[e][j][k] += sum_t T_t[j][k] * p_t with T_t pre-evaluated tables and p_t
 * products of scalars (preeval.cpp:279-451): a generated kernel evaluates the
 * p_t per cell and a DMMA GEMM contracts them with the tables (different
 * summation order: within rounding of the emitted C, not bit-identical).  AUTO
 * takes it when the nest has >= 2048 multiply-adds per cell.
 * ------------------------------------------------------------------------- */
typedef struct femgpu_ir femgpu_ir;

enum {
  FEMGPU_IR_AUTO = 0,
  FEMGPU_IR_THREAD_PER_CELL = 1,
  FEMGPU_IR_WARP_PER_CELL = 2,
  FEMGPU_IR_GEMM = 3
};

typedef struct {
  int noutputs, ninputs, nconstants;
  int per_cell;  /* 1: the nest has an order-free element loop (ncells applies) */
  int strategy;  /* FEMGPU_IR_THREAD_PER_CELL, FEMGPU_IR_WARP_PER_CELL or FEMGPU_IR_GEMM */
} femgpu_ir_info;

/* Parse, generate and compile (FEMGPU_ERR_NOT_FEM_NEST for an IR it cannot
 * emit, FEMGPU_ERR_CUDA if NVRTC is missing or rejects the source). */
int femgpu_ir_create(const char* ir_json, int strategy, femgpu_ir** out);
void femgpu_ir_free(femgpu_ir* k);
int femgpu_ir_get_info(const femgpu_ir* k, femgpu_ir_info* info);
/* Names (group 0 outputs, 1 input tables, 2 constants) and element counts
 * (group 0/1) of the arguments for ncells cells. */
int femgpu_ir_argname(const femgpu_ir* k, int group, int index, char* buf, size_t len);
int femgpu_ir_arg_size(const femgpu_ir* k, int group, int index, long ncells, long* size);
/* The generated CUDA source. */
const char* femgpu_ir_source(const femgpu_ir* k);
/* Device pointers, emit_c order; outputs += ; ncells replaces the IR's extent
 * of the element index. */
int femgpu_ir_launch(femgpu_ir* k, long ncells, double* const* outputs,
                     const double* const* inputs, const double* constants, void* stream);
/* Host pointers, emit_c's calling convention (synchronous). */
int femgpu_ir_argv(femgpu_ir* k, long ncells, double* const* o, const double* const* t,
                   const double* c);

/* The element matrices straight into the global CSR matrix:
 * vals[pos[e][j][k]] += A_e[j][k] (pos from femgpu_csr_positions).  Fused into
 * the element kernel's epilogue where that is faster (P1 Helmholtz: A_e never
 * goes to HBM), else the element kernel into a form-owned scratch (~256 MiB chunks)
 * followed by femgpu_scatter_add.  Device pointers; pos 16-byte aligned.
 * Callers on several streams may share one form: the scratch is handed from
 * one call's last scatter to the next call's stream by an event. */
int femgpu_assemble_csr(const femgpu_form* f, long ncells, const double* coords,
                        const double* coeffs, const long* pos, double* vals, void* stream);

/* Message for the most recent failure on this thread ("" if none). */
const char* femgpu_last_error(void);

/* Library build string (arch, version). */
const char* femgpu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FEMGPU_H */
