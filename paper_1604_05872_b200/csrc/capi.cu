// capi.cu -- the femgpu C ABI (include/femgpu.h): form handles, host-side
// pre-evaluation of reference tensors, dispatch to the sm_100a kernels,
// the host-memory end-to-end pipeline and the emitted-C argv entry point.
//
// Conventions follow libfemopt (proj/src/capi.cpp): thread-local last error
// (:13), exceptions caught at the boundary and mapped to int codes (:15-46).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/femgpu.h"
#include "femgpu_internal.h"

namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    int code = (e == cudaErrorNoDevice || e == cudaErrorNoKernelImageForDevice ||
                e == cudaErrorInsufficientDriver)
                   ? FEMGPU_ERR_NO_DEVICE
                   : FEMGPU_ERR_CUDA;
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_last_error.clear();
    return FEMGPU_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return FEMGPU_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FEMGPU_ERR_INTERNAL;
  }
}

enum Route {
  ROUTE_HELM_P1,
  ROUTE_HELM_TENSOR,
  ROUTE_HELM_QUAD,
  ROUTE_PAIR,
  ROUTE_ELAS_TENSOR,
  ROUTE_BURGERS,
  ROUTE_SVK_MMA,
  ROUTE_BURGERS_QUAD
};

std::string two(int m) {
  char b[8];
  std::snprintf(b, sizeof b, "%02d", m);
  return b;
}

}  // namespace

struct femgpu_form {
  int kind = 0, nq = 0, ns = 0, nc = 0, n = 0, ncoef = 0;
  int schedule = 0, route = 0, device = 0;
  double consts[4] = {0, 0, 0, 0};
  std::vector<double> W, B, D, P;
  femgpu::HelmP1Params p1{};
  double* d_tab = nullptr;
  size_t tab_doubles = 0;
  std::vector<double> h_tab;  // host copy of d_tab (kernels that take tables as parameters)
  double* d_vtab = nullptr;  // element-vector tables (femgpu_assemble_vector), if supported
  double flops_per_cell = 0;
  int kernels_per_launch = 1;
  std::string kernel_name;
  std::vector<std::string> argv_out, argv_tab, argv_con;
  // host-path pipeline resources, created on first use and reused
  static constexpr int NSTREAM = 3;
  std::mutex host_mu;
  cudaStream_t host_st[NSTREAM] = {nullptr, nullptr, nullptr};
  double* host_buf[NSTREAM] = {nullptr, nullptr, nullptr};
  long host_chunk = 0;
  // scratch element matrices for femgpu_assemble_csr on routes without a fused epilogue
  std::mutex csr_mu;
  double* csr_scratch = nullptr;
  long csr_chunk = 0;
  cudaEvent_t csr_done = nullptr;  // recorded after the last scatter that read the scratch

  ~femgpu_form() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (d_tab) cudaFree(d_tab);
    if (d_vtab) cudaFree(d_vtab);
    if (csr_scratch) cudaFree(csr_scratch);
    if (csr_done) cudaEventDestroy(csr_done);
    for (int i = 0; i < NSTREAM; ++i) {
      if (host_buf[i]) cudaFree(host_buf[i]);
      if (host_st[i]) cudaStreamDestroy(host_st[i]);
    }
    cudaSetDevice(cur);
  }
};

namespace {

// ---------------------------------------------------------------------------
// Host pre-evaluation (the reference's symbolic_reduce, preeval.cpp:190-277:
// tables summed over the reduction index in ascending order).
// ---------------------------------------------------------------------------

double Dv(const femgpu_form* f, int a, int q, int j) {
  return f->D[((size_t)a * f->nq + q) * f->ns + j];
}

void build_helm_p1(femgpu_form* f) {
  auto& p = f->p1;
  std::memset(&p, 0, sizeof p);
  for (int m = 0; m < f->nc; ++m) {
    double s = 0.0;
    for (int q = 0; q < f->nq; ++q) s += f->W[q] * f->P[(size_t)q * f->nc + m];
    p.c[m] = s;
    int pp = 0;
    for (int j = 0; j < 4; ++j)
      for (int k = j; k < 4; ++k, ++pp) {
        double t = 0.0;
        for (int q = 0; q < f->nq; ++q)
          t += f->W[q] * f->P[(size_t)q * f->nc + m] * f->B[(size_t)q * 4 + j] * f->B[(size_t)q * 4 + k];
        p.M[m][pp] = t;
      }
  }
  for (int j = 0; j < 4; ++j)
    for (int a = 0; a < 3; ++a) p.Dr[j][a] = Dv(f, a, 0, j);
}

void build_helm_tensor(femgpu_form* f, std::vector<double>& host) {
  int KS, NT, KR, NP;
  femgpu::helm_tensor_geometry(f->ns, f->nc, &KS, &NT, &KR, &NP);
  const int ns = f->ns, nc = f->nc, Q = f->nq;
  // S[alpha = m*7+s][p = (j<=k)]
  std::vector<double> S((size_t)KR * NP, 0.0);
  const int ab[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
  std::vector<double> wp(Q);
  for (int m = 0; m < nc; ++m) {
    for (int q = 0; q < Q; ++q) wp[q] = f->W[q] * f->P[(size_t)q * nc + m];
    int p = 0;
    for (int j = 0; j < ns; ++j)
      for (int k = j; k < ns; ++k, ++p) {
        for (int s = 0; s < 7; ++s) {
          double acc = 0.0;
          for (int q = 0; q < Q; ++q) {
            double v;
            if (s == 6) {
              v = f->B[(size_t)q * ns + j] * f->B[(size_t)q * ns + k];
            } else {
              const int a = ab[s][0], b = ab[s][1];
              v = Dv(f, a, q, j) * Dv(f, b, q, k);
              if (a != b) v += Dv(f, b, q, j) * Dv(f, a, q, k);
            }
            acc += wp[q] * v;
          }
          S[(size_t)(m * 7 + s) * NP + p] = acc;
        }
      }
  }
  host.assign((size_t)KS * NT * 64, 0.0);
  for (int ks = 0; ks < KS; ++ks)
    for (int nt = 0; nt < NT; ++nt)
      for (int lane = 0; lane < 32; ++lane)
        for (int v = 0; v < 2; ++v) {
          const int g = lane >> 2, t = lane & 3;
          const int k = ks * 8 + t + 4 * v, n = nt * 8 + g;
          host[((size_t)(ks * NT + nt) * 32 + lane) * 2 + v] =
              (k < KR && n < NP) ? S[(size_t)k * NP + n] : 0.0;
        }
}

void build_argv_names(femgpu_form* f) {
  auto& T = f->argv_tab;
  T.clear();
  f->argv_out.clear();
  f->argv_con.clear();
  for (int v = 0; v < 4; ++v)
    for (int c = 0; c < 3; ++c) T.push_back("x" + std::to_string(v) + std::to_string(c));
  T.push_back("W");
  const int ns = f->ns;
  switch (f->kind) {
    case FEMGPU_HELMHOLTZ:
      T.push_back("B");
      for (int a = 0; a < 3; ++a) T.push_back("D" + std::to_string(a));
      for (int m = 0; m < f->nc; ++m) {
        T.push_back("P" + two(m));
        T.push_back("f" + two(m));
      }
      f->argv_out.push_back("A");
      break;
    case FEMGPU_ELASTICITY:
    case FEMGPU_HYPERELASTICITY:
      for (int c = 0; c < 3; ++c)
        for (int a = 0; a < 3; ++a) T.push_back("Dv" + std::to_string(c) + std::to_string(a));
      for (int m = 0; m < 4; ++m) {
        T.push_back("P" + std::to_string(m));
        T.push_back("mu" + std::to_string(m));
        T.push_back("lam" + std::to_string(m));
      }
      if (f->kind == FEMGPU_HYPERELASTICITY)
        for (int m = 0; m < ns; ++m)
          for (int a = 0; a < 3; ++a) {
            T.push_back("Dw" + std::to_string(a) + two(m));
            T.push_back("w" + std::to_string(a) + two(m));
          }
      f->argv_out.push_back("A");
      break;
    case FEMGPU_BURGERS:
      T.push_back("B");
      for (int a = 0; a < 3; ++a) T.push_back("D" + std::to_string(a));
      for (int m = 0; m < ns; ++m) {
        T.push_back("P" + two(m));
        for (int a = 0; a < 3; ++a) {
          T.push_back("Du" + std::to_string(a) + two(m));
          T.push_back("u" + std::to_string(a) + two(m));
        }
      }
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) f->argv_out.push_back("A" + std::to_string(c) + std::to_string(d));
      f->argv_con = {"dt", "nu"};
      break;
  }
  std::sort(T.begin(), T.end());
  std::sort(f->argv_out.begin(), f->argv_out.end());
  std::sort(f->argv_con.begin(), f->argv_con.end());
}

// Column of cell-major coeffs that IR e-table `name` maps to, or -1.
int coef_column(const femgpu_form* f, const std::string& name) {
  const int ns = f->ns;
  auto num = [&](size_t from) { return std::atoi(name.c_str() + from); };
  switch (f->kind) {
    case FEMGPU_HELMHOLTZ:
      if (name.size() == 3 && name[0] == 'f') return num(1);
      break;
    case FEMGPU_ELASTICITY:
      if (name.rfind("mu", 0) == 0) return num(2);
      if (name.rfind("lam", 0) == 0) return 4 + num(3);
      break;
    case FEMGPU_HYPERELASTICITY:
      if (name.rfind("mu", 0) == 0) return 3 * ns + num(2);
      if (name.rfind("lam", 0) == 0) return 3 * ns + 4 + num(3);
      if (name[0] == 'w' && name.size() == 4) return (name[1] - '0') * ns + num(2);
      break;
    case FEMGPU_BURGERS:
      if (name[0] == 'u' && name.size() == 4) return (name[1] - '0') * ns + num(2);
      break;
  }
  return -1;
}

// Values of the reference (non-e) input table `name` as the form's IR defines it
// (paper_1604_05872_b200/ir.py: W, B, D_a, per-dof P / Du / Dw columns, padded
// Dv_ca), from the tables the form was created with.  False for e-tables.
bool expected_table(const femgpu_form* f, const std::string& name, std::vector<double>& v) {
  const int Q = f->nq, ns = f->ns;
  auto num = [&](size_t from) { return std::atoi(name.c_str() + from); };
  auto column = [&](const std::vector<double>& T, size_t off, int ncol, int col) {
    v.resize(Q);
    for (int q = 0; q < Q; ++q) v[q] = T[off + (size_t)q * ncol + col];
  };
  v.clear();
  if (name == "W") {
    v = f->W;
    return true;
  }
  if (name == "B" && (f->kind == FEMGPU_HELMHOLTZ || f->kind == FEMGPU_BURGERS)) {
    v = f->B;
    return true;
  }
  if (name.size() == 2 && name[0] == 'D' && (f->kind == FEMGPU_HELMHOLTZ || f->kind == FEMGPU_BURGERS)) {
    const int a = name[1] - '0';
    v.assign(f->D.begin() + (size_t)a * Q * ns, f->D.begin() + (size_t)(a + 1) * Q * ns);
    return true;
  }
  if (name[0] == 'P') {
    const int m = num(1);
    if (f->kind == FEMGPU_BURGERS)
      column(f->B, 0, ns, m);  // u's basis is the trial space's
    else
      column(f->P, 0, f->nc, m);
    return true;
  }
  if (name.size() == 4 && name.rfind("Dv", 0) == 0) {  // component-padded [Q][3 ns]
    const int c = name[2] - '0', a = name[3] - '0';
    v.assign((size_t)Q * 3 * ns, 0.0);
    for (int q = 0; q < Q; ++q)
      for (int j = 0; j < ns; ++j) v[(size_t)q * 3 * ns + c * ns + j] = Dv(f, a, q, j);
    return true;
  }
  if (name.size() == 5 && (name.rfind("Dw", 0) == 0 || name.rfind("Du", 0) == 0)) {
    const int a = name[2] - '0', m = num(3);
    column(f->D, (size_t)a * Q * ns, ns, m);
    return true;
  }
  return false;
}

void validate(const femgpu_form_desc* d) {
  if (!d) throw Error(FEMGPU_ERR_INVALID_ARG, "null form descriptor");
  if (d->kind < FEMGPU_HELMHOLTZ || d->kind > FEMGPU_BURGERS)
    throw Error(FEMGPU_ERR_INVALID_ARG, "unknown form kind " + std::to_string(d->kind));
  if (d->nq <= 0 || d->ns <= 0 || d->nc < 0)
    throw Error(FEMGPU_ERR_INCONSISTENT_LAYOUT, "non-positive table extent");
  if (!d->W || !d->B || !d->D || (d->nc > 0 && !d->P))
    throw Error(FEMGPU_ERR_INVALID_ARG, "null reference table");
  if ((d->kind == FEMGPU_ELASTICITY || d->kind == FEMGPU_HYPERELASTICITY) && d->nc != 4)
    throw Error(FEMGPU_ERR_INCONSISTENT_LAYOUT, "mu and lambda must be P1 (nc == 4)");
  if (d->kind == FEMGPU_BURGERS && !(d->consts[1] != 0.0))
    throw Error(FEMGPU_ERR_INVALID_ARG, "Burgers needs dt != 0 (consts[1])");
  if (d->schedule < FEMGPU_SCHED_AUTO || d->schedule > FEMGPU_SCHED_QUADRATURE_MMA)
    throw Error(FEMGPU_ERR_INVALID_ARG, "unknown schedule");
}

bool constant_gradients(const femgpu_form_desc* d) {
  for (int a = 0; a < 3; ++a)
    for (int q = 1; q < d->nq; ++q)
      for (int j = 0; j < d->ns; ++j)
        if (d->D[((size_t)a * d->nq + q) * d->ns + j] != d->D[((size_t)a * d->nq) * d->ns + j])
          return false;
  return true;
}

// ---------------------------------------------------------------------------
// Schedule choice.  Every kernel that supports a form is a candidate with the
// FP64 flops it executes and the compulsory bytes it moves per cell; its
// predicted time is the roofline time on the current device divided by the
// fraction of the roofline the kernel was measured to reach on B200 at the
// BASELINE sizes (tools/sched_compare.py -> profiles/schedule_choice_r02.json,
// nominal peaks from the device attributes).  The reference makes the same
// choice per monomial from its own flop counts (theta_pre vs theta_se,
// cost.cpp:61-116; plan search driver.cpp:47-106); on the GPU bytes and the
// FP64 pipe's rate enter too, so a 5x flop advantage of the tensor schedule
// (P3 Helmholtz) and an HBM tie between two elasticity schedules are both
// decided by time.
// ---------------------------------------------------------------------------
struct Cand {
  int route, schedule, pipe;
  double flops, eff;
  std::string name;
};

struct Peaks {
  double flops, bytes;
};

Peaks device_peaks() {
  int dev = 0, sms = 148, clk = 1965000, mclk = 3996000, bus = 8192;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrClockRate, dev) == cudaSuccess && v > 0) clk = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMemoryClockRate, dev) == cudaSuccess && v > 0) mclk = v;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrGlobalMemoryBusWidth, dev) == cudaSuccess && v > 0) bus = v;
  }
  // 64 FP64 FMA lanes per SM per clock (DFMA and DMMA alike on B200); DDR HBM
  return {(double)sms * clk * 1e3 * 128.0, 2.0 * mclk * 1e3 * bus / 8.0};
}

// Measured fraction of the nominal roofline per kernel (B200 at 1965 MHz, nominal
// 37.2 TFLOP/s FP64 and 7.67 TB/s from the device attributes; BASELINE meshes;
// profiles/schedule_choice_r02.json, tools/sched_compare.py).  The quadrature
// Helmholtz kernel maps one warp per 4x4 (j,k) tile: ns = 4 keeps one of 16 warps busy.
constexpr double kEffHelmP1 = 0.831, kEffHelmTensor = 0.754, kEffPairElas = 0.726,
                 kEffElasTensor = 0.381, kEffPairSvk = 0.524, kEffBurgers = 0.589,
                 kEffSvkMma = 0.458, kEffBurgersQuad = 0.236;
double eff_helm_quad(int ns) { return ns >= 20 ? 0.245 : ns >= 10 ? 0.2 : 0.04; }

std::vector<Cand> candidates(const femgpu_form_desc* d) {
  std::vector<Cand> c;
  const int Q = d->nq, ns = d->ns, nc = d->nc;
  switch (d->kind) {
    case FEMGPU_HELMHOLTZ:
      if (ns == 4 && nc == 4 && constant_gradients(d))
        // geometry ~60 + gradients 36*2 + mass/combine 8 + stiffness 10 pairs x (5+8+3)
        c.push_back({ROUTE_HELM_P1, FEMGPU_SCHED_TENSOR, 0, 60 + 72 + 8 + 10 * (5 + 8 + 3.0),
                     kEffHelmP1, "helm_p1_kernel"});
      if (femgpu::helm_tensor_supported(ns, nc)) {
        int KS, NT, KR, NP;
        femgpu::helm_tensor_geometry(ns, nc, &KS, &NT, &KR, &NP);
        c.push_back({ROUTE_HELM_TENSOR, FEMGPU_SCHED_TENSOR, 1, 2.0 * KR * NP + 60 + 36 + KR,
                     kEffHelmTensor, "helm_tensor_kernel"});
      }
      if (femgpu::helm_quad_supported(ns, nc)) {
        // per point: f (2 nc), s (2), records 15 ns, j-side scaling 4 ns, pairs 8 (j<=k)
        const double per_q = 2.0 * nc + 2 + 15.0 * ns + 4.0 * ns + 8.0 * ns * (ns + 1) / 2;
        c.push_back({ROUTE_HELM_QUAD, FEMGPU_SCHED_QUADRATURE, 0, 60 + Q * per_q,
                     eff_helm_quad(ns), "helm_quad_kernel"});
      }
      break;
    case FEMGPU_ELASTICITY:
      if (femgpu::pair_supported(d->kind, Q, ns))
        c.push_back({ROUTE_PAIR, FEMGPU_SCHED_QUADRATURE, 0,
                     60 + Q * (ns * 3 * 5 + 16 + ns * (ns + 1) / 2 * 24.0 * 2), kEffPairElas,
                     "pair_ws_kernel"});
      if (femgpu::elas_tensor_supported(ns, nc))
        // alpha: 6 blocks x 36 x 3; GEMM: 3 full 10x10 + 3 upper halves (55) x 36 x 2
        c.push_back({ROUTE_ELAS_TENSOR, FEMGPU_SCHED_TENSOR, 1,
                     60 + 6.0 * 36 * 3 + 2.0 * 36 * (3 * 100 + 3 * 55), kEffElasTensor,
                     "elas_tensor_kernel"});
      break;
    case FEMGPU_HYPERELASTICITY:
      if (femgpu::pair_supported(d->kind, Q, ns)) {
        // per point: setup (coefficients, F, tr E, F F^T, g_j, h_j ~ 340 FMA); per (j,k)
        // 2x2 tile 126 FP64 instructions off the diagonal, 87 on it
        const int nj = ns / 2;
        c.push_back({ROUTE_PAIR, FEMGPU_SCHED_QUADRATURE, 0,
                     60 + Q * 2.0 * (340 + nj * (nj - 1) / 2 * 126 + nj * 87), kEffPairSvk,
                     "pair_svk_ws_kernel"});
      }
      if (femgpu::svk_mma_supported(Q, ns))
        // per point: setup (coefficients, F, tr E, m_cd ~ 160), g_j, h_j (2 x 90) and the
        // 55 G_jk (165) as FMAs; per 4-point stage 27 DMMA.8x8x4 (Ylam, Ymu upper tiles, W)
        c.push_back({ROUTE_SVK_MMA, FEMGPU_SCHED_QUADRATURE_MMA, 1,
                     60 + Q * 2.0 * (160 + 180 + 165) + (Q + 3) / 4 * 27 * 512.0, kEffSvkMma,
                     "svk_mma_kernel"});
      break;
    case FEMGPU_BURGERS:
      if (femgpu::burgers_supported(Q, ns)) {
        const double r = 10;  // derivative-space rank of P3 (checked when the tables are built)
        // g^{cd}: 3c x 3a x r x 20 + 9 x r x 3; GEMM-1: 9 (c,d) x r x 210 (j<=k);
        // GEMM-2: 67 x 400; geometry + GEMM-2 A
        c.push_back({ROUTE_BURGERS, FEMGPU_SCHED_TENSOR, 1,
                     2.0 * 9 * r * 20 + 2.0 * 9 * r * 3 + 2.0 * 9 * r * 210 + 2.0 * 67 * 400 +
                         60 * 7 + 60,
                     kEffBurgers, "burgers_kernel"});
      }
      if (femgpu::burgers_quad_supported(Q, ns))
        // per point: u, grad u (420 FMA, once per cell); per (j, k): g_k (9, per lane
        // and j group), the nine d_d u_c sums (9) and the scalar term (~6)
        c.push_back({ROUTE_BURGERS_QUAD, FEMGPU_SCHED_QUADRATURE, 0,
                     2.0 * Q * (420 + ns / 4 * ns * 12 + (double)ns * ns * 16), kEffBurgersQuad,
                     "burgers_quad_kernel"});
      break;
  }
  return c;
}

double bytes_per_cell(const femgpu_form_desc* d) {
  const int n = d->kind == FEMGPU_HELMHOLTZ ? d->ns : 3 * d->ns;
  const int ncoef = d->kind == FEMGPU_HELMHOLTZ       ? d->nc
                    : d->kind == FEMGPU_ELASTICITY      ? 8
                    : d->kind == FEMGPU_HYPERELASTICITY ? 3 * d->ns + 8
                                                       : 3 * d->ns;
  return 8.0 * (12 + ncoef + (double)n * n);
}

double predicted_ns(const Cand& c, double bytes, const Peaks& pk) {
  return std::max(c.flops / pk.flops, bytes / pk.bytes) / c.eff * 1e9;
}

// Candidates ranked by predicted time; index of the one `schedule` selects, or -1.
int rank_schedules(const femgpu_form_desc* d, std::vector<Cand>& c) {
  c = candidates(d);
  const Peaks pk = device_peaks();
  const double b = bytes_per_cell(d);
  std::stable_sort(c.begin(), c.end(), [&](const Cand& x, const Cand& y) {
    const double tx = predicted_ns(x, b, pk), ty = predicted_ns(y, b, pk);
    return tx != ty ? tx < ty : x.flops < y.flops;
  });
  for (size_t i = 0; i < c.size(); ++i)
    if (d->schedule == FEMGPU_SCHED_AUTO || d->schedule == c[i].schedule) return (int)i;
  return -1;
}

void check_ptr(const void* p, const char* what) {
  if (!p) throw Error(FEMGPU_ERR_INVALID_ARG, std::string("null ") + what);
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
    throw Error(FEMGPU_ERR_INVALID_ARG, std::string(what) + " must be 16-byte aligned");
}

void launch(const femgpu_form* f, long E, const double* coords, const double* coef, double* A,
            int acc, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  switch (f->route) {
    case ROUTE_HELM_P1:
      e = femgpu::launch_helm_p1(f->p1, E, coords, coef, A, acc, s);
      break;
    case ROUTE_HELM_TENSOR:
      e = femgpu::launch_helm_tensor(f->ns, f->nc, E, coords, coef, f->d_tab, A, acc, s);
      break;
    case ROUTE_HELM_QUAD:
      e = femgpu::launch_helm_quad(f->ns, f->nq, f->nc, E, coords, coef, f->d_tab, A, acc, s);
      break;
    case ROUTE_PAIR:
      e = femgpu::launch_pair(f->kind, f->nq, f->ns, E, coords, coef, f->d_tab, f->h_tab.data(),
                              A, acc, s);
      break;
    case ROUTE_ELAS_TENSOR:
      e = femgpu::launch_elas_tensor(E, coords, coef, f->d_tab, A, acc, s);
      break;
    case ROUTE_SVK_MMA:
      e = femgpu::launch_svk_mma(f->nq, f->ns, E, coords, coef, f->d_tab, A, acc, s);
      break;
    case ROUTE_BURGERS_QUAD:
      e = femgpu::launch_burgers_quad(f->nq, f->ns, E, coords, coef, f->d_tab, f->consts[0],
                                      f->consts[1], A, acc, s);
      break;
    case ROUTE_BURGERS:
      e = femgpu::launch_burgers(f->ns, E, coords, coef, f->d_tab, f->consts[0], f->consts[1], A,
                                 acc, s);
      break;
  }
  cuda_check(e, f->kernel_name.c_str());
}

}  // namespace

namespace femgpu {
void set_last_error(const std::string& m) { g_last_error = m; }

cudaError_t once_per_device(const void* key, const std::function<cudaError_t()>& init) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  const cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({key, dev})) return cudaSuccess;
  const cudaError_t r = init();
  if (r == cudaSuccess) done.insert({key, dev});
  return r;
}
}  // namespace femgpu

extern "C" {

int femgpu_form_create(const femgpu_form_desc* d, femgpu_form** out) {
  if (!out) {
    g_last_error = "null output handle";
    return FEMGPU_ERR_INVALID_ARG;
  }
  *out = nullptr;
  return guarded([&] {
    validate(d);
    auto f = std::make_unique<femgpu_form>();
    f->kind = d->kind;
    f->nq = d->nq;
    f->ns = d->ns;
    f->nc = d->nc;
    f->n = d->kind == FEMGPU_HELMHOLTZ ? d->ns : 3 * d->ns;
    f->ncoef = d->kind == FEMGPU_HELMHOLTZ      ? d->nc
               : d->kind == FEMGPU_ELASTICITY   ? 8
               : d->kind == FEMGPU_HYPERELASTICITY ? 3 * d->ns + 8
                                               : 3 * d->ns;
    std::memcpy(f->consts, d->consts, sizeof f->consts);
    f->W.assign(d->W, d->W + d->nq);
    f->B.assign(d->B, d->B + (size_t)d->nq * d->ns);
    f->D.assign(d->D, d->D + (size_t)3 * d->nq * d->ns);
    if (d->nc > 0) f->P.assign(d->P, d->P + (size_t)d->nq * d->nc);
    cuda_check(cudaGetDevice(&f->device), "cudaGetDevice");
    std::vector<double> host;
    std::vector<Cand> cands;
    const int pick = rank_schedules(d, cands);
    if (pick < 0)
      throw Error(FEMGPU_ERR_UNSUPPORTED,
                  cands.empty() ? "no kernel for this form's sizes"
                                : "no kernel of the requested schedule for this form");
    const Cand& ch = cands[pick];
    f->route = ch.route;
    f->schedule = ch.schedule;
    f->flops_per_cell = ch.flops;
    f->kernel_name = ch.name;
    switch (ch.route) {
      case ROUTE_HELM_P1:
        build_helm_p1(f.get());
        break;
      case ROUTE_HELM_TENSOR:
        build_helm_tensor(f.get(), host);
        break;
      case ROUTE_BURGERS_QUAD:  // W | B | D
        host.insert(host.end(), f->W.begin(), f->W.end());
        host.insert(host.end(), f->B.begin(), f->B.end());
        host.insert(host.end(), f->D.begin(), f->D.end());
        break;
      case ROUTE_HELM_QUAD:  // W | B | D | P
        host.insert(host.end(), f->W.begin(), f->W.end());
        host.insert(host.end(), f->B.begin(), f->B.end());
        host.insert(host.end(), f->D.begin(), f->D.end());
        host.insert(host.end(), f->P.begin(), f->P.end());
        break;
      case ROUTE_ELAS_TENSOR:
        host.assign(femgpu::elas_tensor_table_doubles(), 0.0);
        femgpu::elas_tensor_tables(f->nq, f->W.data(), f->D.data(), f->P.data(), host.data());
        break;
      case ROUTE_PAIR:  // W | D | P
      case ROUTE_SVK_MMA:
        host.insert(host.end(), f->W.begin(), f->W.end());
        host.insert(host.end(), f->D.begin(), f->D.end());
        host.insert(host.end(), f->P.begin(), f->P.end());
        break;
      case ROUTE_BURGERS:
        host.assign(femgpu::burgers_table_doubles(), 0.0);
        if (femgpu::burgers_tables(f->nq, f->W.data(), f->B.data(), f->D.data(), host.data()) < 0)
          throw Error(FEMGPU_ERR_UNSUPPORTED,
                      "Burgers kernel: derivative tables do not span a space of rank <= 12");
        break;
    }
    if (!host.empty()) {
      f->tab_doubles = host.size();
      f->h_tab = host;
      cuda_check(cudaMalloc(&f->d_tab, host.size() * sizeof(double)), "cudaMalloc(tables)");
      cuda_check(cudaMemcpy(f->d_tab, host.data(), host.size() * sizeof(double),
                            cudaMemcpyHostToDevice),
                 "cudaMemcpy(tables)");
    }
    if (femgpu::vector_supported(f->kind, f->ns, f->nc)) {
      // element-vector tables (vector.cu): Helmholtz M_jm = sum_q W_q B_qj P_qm (ascending
      // q, preeval.cpp:269-274); SVK W | D | P; Burgers W | B | D_a (padded, vector.cu)
      std::vector<double> v;
      const int Q = f->nq, ns = f->ns, nc = f->nc;
      if (f->kind == FEMGPU_HELMHOLTZ) {
        v.assign((size_t)ns * nc, 0.0);
        for (int j = 0; j < ns; ++j)
          for (int m = 0; m < nc; ++m) {
            double s = 0.0;
            for (int q = 0; q < Q; ++q)
              s += f->W[q] * f->B[(size_t)q * ns + j] * f->P[(size_t)q * nc + m];
            v[(size_t)j * nc + m] = s;
          }
      } else if (f->kind == FEMGPU_HYPERELASTICITY) {
        v.insert(v.end(), f->W.begin(), f->W.end());
        v.insert(v.end(), f->D.begin(), f->D.end());
        v.insert(v.end(), f->P.begin(), f->P.end());
      } else {  // W[Qp] | T[4][Qp][ns], T_0 = B, T_{1+a} = D_a, zero rows past Q
        const int Qp = femgpu::vector_table_qpad(Q);
        v.assign((size_t)Qp + 4 * (size_t)Qp * ns, 0.0);
        for (int q = 0; q < Q; ++q) {
          v[q] = f->W[q];
          for (int j = 0; j < ns; ++j) {
            v[Qp + (size_t)q * ns + j] = f->B[(size_t)q * ns + j];
            for (int a = 0; a < 3; ++a)
              v[Qp + ((size_t)(1 + a) * Qp + q) * ns + j] = f->D[((size_t)a * Q + q) * ns + j];
          }
        }
      }
      cuda_check(cudaMalloc(&f->d_vtab, v.size() * sizeof(double)), "cudaMalloc(vector tables)");
      cuda_check(cudaMemcpy(f->d_vtab, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice),
                 "cudaMemcpy(vector tables)");
    }
    build_argv_names(f.get());
    *out = f.release();
  });
}

void femgpu_form_free(femgpu_form* f) { delete f; }

int femgpu_form_schedules(const femgpu_form_desc* d, femgpu_schedule_info* out, int cap,
                          int* count) {
  if (!count || (cap > 0 && !out)) {
    g_last_error = "null argument";
    return FEMGPU_ERR_INVALID_ARG;
  }
  return guarded([&] {
    validate(d);
    std::vector<Cand> c;
    const int pick = rank_schedules(d, c);
    const Peaks pk = device_peaks();
    const double b = bytes_per_cell(d);
    *count = (int)c.size();
    for (int i = 0; i < (int)c.size() && i < cap; ++i) {
      femgpu_schedule_info& o = out[i];
      std::memset(&o, 0, sizeof o);
      std::snprintf(o.kernel_name, sizeof o.kernel_name, "%s", c[i].name.c_str());
      o.schedule = c[i].schedule;
      o.pipe = c[i].pipe;
      o.flops_per_cell = c[i].flops;
      o.bytes_per_cell = b;
      o.peak_flops = pk.flops;
      o.peak_bytes = pk.bytes;
      o.efficiency = c[i].eff;
      o.predicted_ns_per_cell = predicted_ns(c[i], b, pk);
      o.chosen = i == pick;
    }
  });
}

int femgpu_form_get_info(const femgpu_form* f, femgpu_form_info* info) {
  if (!f || !info) {
    g_last_error = "null argument";
    return FEMGPU_ERR_INVALID_ARG;
  }
  return guarded([&] {
    std::memset(info, 0, sizeof *info);
    info->n = f->n;
    info->ncoef = f->ncoef;
    info->schedule = f->schedule;
    info->flops_per_cell = f->flops_per_cell;
    info->bytes_per_cell = 8.0 * (12 + f->ncoef + (double)f->n * f->n);
    info->kernels_per_launch = f->kernels_per_launch;
    std::snprintf(info->kernel_name, sizeof info->kernel_name, "%s", f->kernel_name.c_str());
  });
}

int femgpu_assemble(const femgpu_form* f, long ncells, const double* coords, const double* coeffs,
                    double* A, int accumulate, void* stream) {
  if (!f) {
    g_last_error = "null form";
    return FEMGPU_ERR_INVALID_ARG;
  }
  return guarded([&] {
    if (ncells < 0) throw Error(FEMGPU_ERR_INVALID_ARG, "negative cell count");
    if (ncells == 0) return;
    check_ptr(coords, "coords");
    check_ptr(A, "A");
    if (f->ncoef > 0) check_ptr(coeffs, "coeffs");
    int cur = 0;  // the form's tables live on the device it was created on
    cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur != f->device) throw Error(FEMGPU_ERR_INVALID_ARG, "form belongs to another device");
    launch(f, ncells, coords, coeffs, A, accumulate, static_cast<cudaStream_t>(stream));
  });
}

int femgpu_assemble_vector(const femgpu_form* f, long ncells, const double* coords,
                           const double* coeffs, double* b, int accumulate, void* stream) {
  if (!f) {
    g_last_error = "null form";
    return FEMGPU_ERR_INVALID_ARG;
  }
  return guarded([&] {
    if (ncells < 0) throw Error(FEMGPU_ERR_INVALID_ARG, "negative cell count");
    if (!f->d_vtab)
      throw Error(FEMGPU_ERR_UNSUPPORTED, "no element-vector kernel for this form");
    if (ncells == 0) return;
    check_ptr(coords, "coords");
    check_ptr(b, "b");
    if (f->ncoef > 0) check_ptr(coeffs, "coeffs");
    int cur = 0;
    cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur != f->device) throw Error(FEMGPU_ERR_INVALID_ARG, "form belongs to another device");
    cuda_check(femgpu::launch_vector(f->kind, f->nq, f->ns, f->nc, ncells, coords, coeffs, f->d_vtab,
                                     f->consts, b, accumulate, static_cast<cudaStream_t>(stream)),
               "element-vector kernel");
  });
}

int femgpu_assemble_host(const femgpu_form* fc, long ncells, const double* coords,
                         const double* coeffs, double* A, int accumulate) {
  if (!fc) {
    g_last_error = "null form";
    return FEMGPU_ERR_INVALID_ARG;
  }
  femgpu_form* f = const_cast<femgpu_form*>(fc);  // pipeline cache only; guarded below
  return guarded([&] {
    if (ncells < 0) throw Error(FEMGPU_ERR_INVALID_ARG, "negative cell count");
    if (ncells == 0) return;
    if (!coords || !A || (f->ncoef > 0 && !coeffs)) throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    int cur = 0;  // the form's tables and pipeline buffers live on its device
    cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur != f->device) throw Error(FEMGPU_ERR_INVALID_ARG, "form belongs to another device");
    std::lock_guard<std::mutex> lock(f->host_mu);
    const size_t nn = (size_t)f->n * f->n;
    // Chunks of at most ~128 MiB of element matrices and at most 1/8 of the
    // call (so small element matrices still get a pipeline: c1's 1.6 M cells
    // were 2 chunks), at least 8192 cells; multiples of 64 cells.  Three
    // streams rotate H2D -> kernel -> D2H so both copy engines stay busy.
    const long by_bytes = std::max<long>(64, (long)((128u << 20) / (nn * 8)) / 64 * 64);
    const long by_count = std::max<long>(8192, (ncells / 8 + 63) / 64 * 64);
    const long chunk = std::min(by_bytes, by_count);
    const size_t per_cell = 12 + f->ncoef + nn;
    if (f->host_chunk != chunk) {
      f->host_chunk = 0;  // a failed re-allocation leaves no stale size behind
      for (int i = 0; i < femgpu_form::NSTREAM; ++i) {
        if (!f->host_st[i])
          cuda_check(cudaStreamCreateWithFlags(&f->host_st[i], cudaStreamNonBlocking),
                     "cudaStreamCreate");
        if (f->host_buf[i]) cudaFree(f->host_buf[i]);
        f->host_buf[i] = nullptr;
        cuda_check(cudaMalloc(&f->host_buf[i], per_cell * chunk * sizeof(double)),
                   "cudaMalloc(chunk)");
      }
      f->host_chunk = chunk;
    }
    long ci = 0;
    for (long c0 = 0; c0 < ncells; c0 += chunk, ++ci) {
      const long E = std::min(chunk, ncells - c0);
      const int s = (int)(ci % femgpu_form::NSTREAM);
      cudaStream_t st = f->host_st[s];
      double* dx = f->host_buf[s];
      double* dA = dx + 12 * chunk;  // 16B aligned: chunk is a multiple of 64
      double* dc = dA + nn * chunk;
      cuda_check(cudaMemcpyAsync(dx, coords + c0 * 12, E * 12 * sizeof(double),
                                 cudaMemcpyHostToDevice, st), "H2D coords");
      if (f->ncoef > 0)
        cuda_check(cudaMemcpyAsync(dc, coeffs + c0 * f->ncoef, E * f->ncoef * sizeof(double),
                                   cudaMemcpyHostToDevice, st), "H2D coeffs");
      if (accumulate)
        cuda_check(cudaMemcpyAsync(dA, A + c0 * nn, E * nn * sizeof(double),
                                   cudaMemcpyHostToDevice, st), "H2D A");
      launch(f, E, dx, dc, dA, accumulate, st);
      cuda_check(cudaMemcpyAsync(A + c0 * nn, dA, E * nn * sizeof(double), cudaMemcpyDeviceToHost,
                                 st), "D2H A");
    }
    for (int i = 0; i < femgpu_form::NSTREAM; ++i)
      cuda_check(cudaStreamSynchronize(f->host_st[i]), "sync");
  });
}

int femgpu_kernel_argc(const femgpu_form* f, int group, int* count) {
  if (!f || !count || group < 0 || group > 2) {
    g_last_error = "bad argument";
    return FEMGPU_ERR_INVALID_ARG;
  }
  *count = (int)(group == 0 ? f->argv_out.size() : group == 1 ? f->argv_tab.size() : f->argv_con.size());
  g_last_error.clear();
  return FEMGPU_OK;
}

int femgpu_kernel_argname(const femgpu_form* f, int group, int index, char* buf, size_t len) {
  if (!f || !buf || group < 0 || group > 2) {
    g_last_error = "bad argument";
    return FEMGPU_ERR_INVALID_ARG;
  }
  const auto& v = group == 0 ? f->argv_out : group == 1 ? f->argv_tab : f->argv_con;
  if (index < 0 || index >= (int)v.size()) {
    g_last_error = "argument index out of range";
    return FEMGPU_ERR_INVALID_ARG;
  }
  std::snprintf(buf, len, "%s", v[index].c_str());
  g_last_error.clear();
  return FEMGPU_OK;
}

int femgpu_kernel_argv(const femgpu_form* f, long ncells, double* const* o, const double* const* t,
                       const double* c) {
  if (!f || !o || !t) {
    g_last_error = "null argument";
    return FEMGPU_ERR_INVALID_ARG;
  }
  return guarded([&] {
    if (ncells <= 0) return;
    const long E = ncells;
    const int ns = f->ns;
    // SoA e-tables -> cell-major (the layout the kernels stream); reference
    // tables must equal the form's (its kernels use the form's own copies)
    std::vector<double> coords((size_t)E * 12), coef((size_t)E * std::max(f->ncoef, 1));
    std::vector<double> want;
    for (size_t i = 0; i < f->argv_tab.size(); ++i) {
      const std::string& name = f->argv_tab[i];
      if (expected_table(f, name, want)) {
        if (!t[i]) throw Error(FEMGPU_ERR_INVALID_ARG, "null table " + name);
        if (std::memcmp(t[i], want.data(), want.size() * sizeof(double)) != 0)
          throw Error(FEMGPU_ERR_INCONSISTENT_LAYOUT,
                      "table " + name + " differs from the form's reference tables");
        continue;
      }
      if (name.size() == 3 && name[0] == 'x') {
        const int v = name[1] - '0', cc = name[2] - '0';
        if (!t[i]) throw Error(FEMGPU_ERR_INVALID_ARG, "null table " + name);
        for (long e = 0; e < E; ++e) coords[e * 12 + v * 3 + cc] = t[i][e];
        continue;
      }
      const int col = coef_column(f, name);
      if (col >= 0) {
        if (!t[i]) throw Error(FEMGPU_ERR_INVALID_ARG, "null table " + name);
        for (long e = 0; e < E; ++e) coef[e * f->ncoef + col] = t[i][e];
      }
    }
    if (f->kind == FEMGPU_BURGERS && c) {
      // constants in name order: dt, nu -- must match the form's
      if (c[0] != f->consts[1] || c[1] != f->consts[0])
        throw Error(FEMGPU_ERR_INCONSISTENT_LAYOUT, "constants differ from the form's (nu, dt)");
    }
    const size_t nn = (size_t)f->n * f->n;
    std::vector<double> A((size_t)E * nn, 0.0);
    int rc = femgpu_assemble_host(f, E, coords.data(), coef.data(), A.data(), 0);
    if (rc != FEMGPU_OK) throw Error(rc, g_last_error);
    if (f->kind == FEMGPU_BURGERS) {
      for (int cc = 0; cc < 3; ++cc)
        for (int d = 0; d < 3; ++d) {
          double* out = o[cc * 3 + d];  // names A00..A22 sorted
          for (long e = 0; e < E; ++e)
            for (int j = 0; j < ns; ++j)
              for (int k = 0; k < ns; ++k)
                out[(e * ns + j) * ns + k] += A[e * nn + (size_t)(cc * ns + j) * f->n + d * ns + k];
        }
    } else {
      for (size_t i = 0; i < A.size(); ++i) o[0][i] += A[i];
    }
  });
}

int femgpu_gather(long ncells, int ncoef, const double* V, const int* cells, const double* coef,
                  const int* coef_idx, double* coords, double* coeffs, void* stream) {
  return guarded([&] {
    if (ncells < 0 || ncoef < 0) throw Error(FEMGPU_ERR_INVALID_ARG, "negative size");
    if (ncells == 0) return;
    if (!V || !cells || !coords || (ncoef > 0 && (!coef || !coef_idx || !coeffs)))
      throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    cuda_check(femgpu::launch_gather(ncells, ncoef, V, cells, coef, coef_idx, coords, coeffs,
                                     static_cast<cudaStream_t>(stream)),
               "gather_kernel");
  });
}

int femgpu_csr_positions(long ncells, int n, const int* dof_map, const long* row_ptr,
                         const int* col_idx, long* pos, void* stream) {
  return guarded([&] {
    if (ncells < 0 || n <= 0) throw Error(FEMGPU_ERR_INVALID_ARG, "bad size");
    if (ncells == 0) return;
    if (!dof_map || !row_ptr || !col_idx || !pos) throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int* d_missing = nullptr;
    cuda_check(cudaMallocAsync(&d_missing, sizeof(int), s), "cudaMallocAsync");
    cuda_check(cudaMemsetAsync(d_missing, 0, sizeof(int), s), "cudaMemsetAsync");
    cudaError_t e = femgpu::launch_csr_positions(ncells, n, dof_map, row_ptr, col_idx, pos,
                                                 d_missing, s);
    int missing = 0;
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&missing, d_missing, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d_missing, s);
    cuda_check(e, "csr_positions_kernel");
    if (missing)
      throw Error(FEMGPU_ERR_INCONSISTENT_LAYOUT,
                  std::to_string(missing) + " element-matrix entries outside the CSR pattern");
  });
}

int femgpu_assemble_csr(const femgpu_form* fc, long ncells, const double* coords,
                        const double* coeffs, const long* pos, double* vals, void* stream) {
  if (!fc) {
    g_last_error = "null form";
    return FEMGPU_ERR_INVALID_ARG;
  }
  femgpu_form* f = const_cast<femgpu_form*>(fc);  // scratch cache only; guarded below
  return guarded([&] {
    if (ncells < 0) throw Error(FEMGPU_ERR_INVALID_ARG, "negative cell count");
    if (ncells == 0) return;
    if (!coords || !pos || !vals || (f->ncoef > 0 && !coeffs))
      throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    check_ptr(coords, "coords");
    if (f->ncoef > 0) check_ptr(coeffs, "coeffs");
    check_ptr(pos, "pos");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int cur = 0;
    cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur != f->device) throw Error(FEMGPU_ERR_INVALID_ARG, "form belongs to another device");
    if (f->route == ROUTE_HELM_P1) {  // fused epilogue: A_e never leaves the SM
      cuda_check(femgpu::launch_helm_p1(f->p1, ncells, coords, coeffs, nullptr, 0, s, pos, vals),
                 f->kernel_name.c_str());
      return;
    }
    // element kernel into a form-owned scratch, then the scatter-add (chunks of
    // ~256 MiB of element matrices).  A fused copy-out in the warp-specialised
    // tensor kernels was measured slower: its 4 IO warps cannot issue the atomics
    // of a 32-cell tile in the time the MMA warps take (c2: 4.5 vs 3.0 ms).
    // One scratch per form, shared by every caller: the lock orders the enqueues
    // and the csr_done event orders the GPU work -- this call's stream waits for
    // the previous call's last scatter (on whatever stream) before overwriting.
    std::lock_guard<std::mutex> lock(f->csr_mu);
    const size_t nn = (size_t)f->n * f->n;
    const long chunk = std::max<long>(64, (long)((256u << 20) / (nn * 8)) / 64 * 64);
    if (!f->csr_done)
      cuda_check(cudaEventCreateWithFlags(&f->csr_done, cudaEventDisableTiming), "cudaEventCreate");
    if (!f->csr_scratch || f->csr_chunk != chunk) {
      cuda_check(cudaEventSynchronize(f->csr_done), "cudaEventSynchronize");
      if (f->csr_scratch) cudaFree(f->csr_scratch);
      f->csr_scratch = nullptr;
      f->csr_chunk = 0;
      cuda_check(cudaMalloc(&f->csr_scratch, chunk * nn * sizeof(double)), "cudaMalloc(scratch)");
      f->csr_chunk = chunk;
    }
    cuda_check(cudaStreamWaitEvent(s, f->csr_done, 0), "cudaStreamWaitEvent");
    for (long c0 = 0; c0 < ncells; c0 += chunk) {
      const long E = std::min(chunk, ncells - c0);
      launch(f, E, coords + c0 * 12, f->ncoef > 0 ? coeffs + c0 * f->ncoef : coeffs,
             f->csr_scratch, 0, s);
      cuda_check(femgpu::launch_scatter_add(E * (long)nn, f->csr_scratch, pos + c0 * (long)nn, vals, s),
                 "scatter_add_kernel");
    }
    cuda_check(cudaEventRecord(f->csr_done, s), "cudaEventRecord");
  });
}

int femgpu_scatter_add(long nentries, const double* A, const long* pos, double* vals,
                       void* stream) {
  return guarded([&] {
    if (nentries < 0) throw Error(FEMGPU_ERR_INVALID_ARG, "negative size");
    if (nentries == 0) return;
    if (!A || !pos || !vals) throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    cuda_check(femgpu::launch_scatter_add(nentries, A, pos, vals, static_cast<cudaStream_t>(stream)),
               "scatter_add_kernel");
  });
}

int femgpu_csr_row_offsets(long ncells, int n, const int* dof_map, const long* row_ptr,
                           const long* pos, uint16_t* loc, void* stream) {
  return guarded([&] {
    if (ncells < 0 || n <= 0) throw Error(FEMGPU_ERR_INVALID_ARG, "bad size");
    if (ncells == 0) return;
    if (!dof_map || !row_ptr || !pos || !loc) throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int* d_bad = nullptr;
    cuda_check(cudaMallocAsync(&d_bad, sizeof(int), s), "cudaMallocAsync");
    cuda_check(cudaMemsetAsync(d_bad, 0, sizeof(int), s), "cudaMemsetAsync");
    cudaError_t e = femgpu::launch_csr_row_offsets(ncells, n, dof_map, row_ptr, pos, loc, d_bad, s);
    int bad = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d_bad, s);
    cuda_check(e, "csr_row_offsets_kernel");
    if (bad)
      throw Error(FEMGPU_ERR_INCONSISTENT_LAYOUT,
                  std::to_string(bad) + " element-matrix entries outside their CSR row");
  });
}

int femgpu_csr_gather_rows(long nrows, int n, const long* row_ptr, const long* inc_ptr,
                           const int* inc, const uint16_t* loc, int max_row_len,
                           const double* A, double* vals, int accumulate, void* stream) {
  return guarded([&] {
    if (nrows < 0 || n <= 0 || n > 64) throw Error(FEMGPU_ERR_INVALID_ARG, "bad size (n <= 64)");
    if (nrows == 0) return;
    if (max_row_len <= 0 || max_row_len > 65536)
      throw Error(FEMGPU_ERR_INVALID_ARG, "max_row_len out of range");
    if (!row_ptr || !inc_ptr || !inc || !loc || !A || !vals)
      throw Error(FEMGPU_ERR_INVALID_ARG, "null buffer");
    cuda_check(femgpu::launch_csr_gather_rows(nrows, n, max_row_len, row_ptr, inc_ptr, inc, loc, A,
                                              accumulate, vals, static_cast<cudaStream_t>(stream)),
               "csr_gather_rows_kernel");
  });
}

const char* femgpu_last_error(void) { return g_last_error.c_str(); }

const char* femgpu_version(void) { return "femgpu 0.1 (sm_100a, FP64)"; }

}  // extern "C"
