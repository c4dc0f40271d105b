/* femoracle.c -- CPU restatement of the element kernels. TEST INFRASTRUCTURE.
 *
 * This is the parity oracle ("port"): plain C, straight quadrature loops, no
 * schedule tricks.  Each form evaluates exactly the integrand of the *raw*
 * (unoptimized) femopt IR that paper_1604_05872_b200/ir.py writes for it,
 * with the reference interpreter's semantics (proj/src/interp.cpp:50-121:
 * outputs zeroed on entry, `+=` accumulation in loop order e, i, j, k).  It is
 * pinned against the reference itself (oracle/_ref: femopt's interpreter and
 * its optimized emitted C) by tests/test_oracle.py on tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it.  The product (libfemgpu.so) never does.
 *
 * Layouts (cell-major FP64, as the C ABI in include/femgpu.h):
 *   coords [E][4][3], coeffs [E][ncoef], A [E][n][n] (overwritten),
 *   W [Q], B [Q][ns], D [3][Q][ns], P [Q][nc] (coefficient basis).
 */
#include <math.h>
#include <stddef.h>
#include <string.h>

enum { HELMHOLTZ = 1, ELASTICITY = 2, HYPERELASTICITY = 3, BURGERS = 4 };

/* Level-1 preheader of the IR (ir.py geometry_statements): J, cofactors,
 * det, rdet = 1/det, adet = |det|, K = J^-1 with K_ab = C_ba * rdet. */
static void geometry(const double* x, double K[3][3], double* adet) {
  double J[3][3], Cf[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) J[a][b] = x[(b + 1) * 3 + a] + (-1.0) * x[a];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      int a1 = a == 0 ? 1 : 0, a2 = a == 2 ? 1 : 2;
      int b1 = b == 0 ? 1 : 0, b2 = b == 2 ? 1 : 2;
      double m = J[a1][b1] * J[a2][b2] + (-1.0) * (J[a1][b2] * J[a2][b1]);
      Cf[a][b] = ((a + b) % 2 == 0) ? m : -m;
    }
  double det = J[0][0] * Cf[0][0] + J[0][1] * Cf[0][1] + J[0][2] * Cf[0][2];
  double rdet = 1.0 / det;
  *adet = fabs(det);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) K[a][b] = Cf[b][a] * rdet;
}

/* Physical gradients g[j][beta] = sum_a K[a][beta] D[a][q][j]. */
static void phys_grad(int Q, int ns, int q, const double* D, double K[3][3], double* g) {
  for (int j = 0; j < ns; ++j)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int a = 0; a < 3; ++a) s += K[a][b] * D[((size_t)a * Q + q) * ns + j];
      g[j * 3 + b] = s;
    }
}

static void cell_helmholtz(int Q, int ns, int nc, const double* W, const double* B,
                           const double* D, const double* P, const double* x,
                           const double* f, double* A) {
  double K[3][3], adet, g[20 * 3];
  geometry(x, K, &adet);
  memset(A, 0, sizeof(double) * ns * ns);
  for (int q = 0; q < Q; ++q) {
    phys_grad(Q, ns, q, D, K, g);
    double fq = 0.0;
    for (int m = 0; m < nc; ++m) fq += f[m] * P[q * nc + m];
    double s = fq * W[q] * adet;
    for (int j = 0; j < ns; ++j)
      for (int k = 0; k < ns; ++k) {
        double st = g[j * 3] * g[k * 3] + g[j * 3 + 1] * g[k * 3 + 1] + g[j * 3 + 2] * g[k * 3 + 2];
        A[j * ns + k] += (st + B[q * ns + j] * B[q * ns + k]) * s;
      }
  }
}

static void cell_elasticity(int Q, int ns, const double* W, const double* D, const double* P,
                            const double* x, const double* cf, double* A) {
  const int n = 3 * ns;
  double K[3][3], adet, g[10 * 3];
  geometry(x, K, &adet);
  memset(A, 0, sizeof(double) * n * n);
  for (int q = 0; q < Q; ++q) {
    phys_grad(Q, ns, q, D, K, g);
    double mu = 0.0, lam = 0.0;
    for (int m = 0; m < 4; ++m) {
      mu += cf[m] * P[q * 4 + m];
      lam += cf[4 + m] * P[q * 4 + m];
    }
    double s = W[q] * adet;
    for (int J = 0; J < n; ++J)
      for (int Kk = 0; Kk < n; ++Kk) {
        int c = J / ns, j = J % ns, d = Kk / ns, k = Kk % ns;
        /* grad v_J (c',b) = delta(c',c) g_j[b]; eps = sym part. */
        double ee = 0.0;
        for (int cc = 0; cc < 3; ++cc)
          for (int b = 0; b < 3; ++b) {
            double ej = 0.5 * ((cc == c ? g[j * 3 + b] : 0.0) + (b == c ? g[j * 3 + cc] : 0.0));
            double ek = 0.5 * ((cc == d ? g[k * 3 + b] : 0.0) + (b == d ? g[k * 3 + cc] : 0.0));
            ee += ej * ek;
          }
        double dd = g[j * 3 + c] * g[k * 3 + d];
        A[J * n + Kk] += (2.0 * mu * ee + lam * dd) * s;
      }
  }
}

static void cell_svk(int Q, int ns, const double* W, const double* D, const double* P,
                     const double* x, const double* cf, double* A) {
  const int n = 3 * ns;
  const double* w = cf;           /* [3][ns] */
  const double* mu_d = cf + 3 * ns;
  const double* lam_d = cf + 3 * ns + 4;
  double K[3][3], adet, g[10 * 3];
  geometry(x, K, &adet);
  memset(A, 0, sizeof(double) * n * n);
  for (int q = 0; q < Q; ++q) {
    phys_grad(Q, ns, q, D, K, g);
    double mu = 0.0, lam = 0.0;
    for (int m = 0; m < 4; ++m) {
      mu += mu_d[m] * P[q * 4 + m];
      lam += lam_d[m] * P[q * 4 + m];
    }
    double F[3][3], E[3][3], S[3][3];
    for (int c = 0; c < 3; ++c)
      for (int b = 0; b < 3; ++b) {
        double gw = 0.0;
        for (int m = 0; m < ns; ++m) gw += w[c * ns + m] * g[m * 3 + b];
        F[c][b] = (c == b ? 1.0 : 0.0) + gw;
      }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double t = F[0][a] * F[0][b] + F[1][a] * F[1][b] + F[2][a] * F[2][b];
        E[a][b] = 0.5 * (a == b ? t - 1.0 : t);
      }
    double trE = E[0][0] + E[1][1] + E[2][2];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) S[a][b] = (a == b ? lam * trE : 0.0) + 2.0 * mu * E[a][b];
    double s = W[q] * adet;
    for (int J = 0; J < n; ++J)
      for (int Kk = 0; Kk < n; ++Kk) {
        int c = J / ns, j = J % ns, d = Kk / ns, k = Kk % ns;
        const double* gj = g + j * 3;
        const double* gk = g + k * 3;
        /* grad du = e_d (x) g_k, grad v = e_c (x) g_j. */
        double trdE = F[d][0] * gk[0] + F[d][1] * gk[1] + F[d][2] * gk[2];
        double tot = 0.0;
        for (int b = 0; b < 3; ++b) {
          double geo = 0.0;
          if (c == d)
            for (int qq = 0; qq < 3; ++qq) geo += gk[qq] * S[qq][b];
          double mat1 = lam * trdE * F[c][b];
          double m2 = 0.0;
          for (int qq = 0; qq < 3; ++qq) m2 += F[c][qq] * (gk[qq] * F[d][b] + F[d][qq] * gk[b]);
          tot += gj[b] * (geo + mat1 + mu * m2);
        }
        A[J * n + Kk] += tot * s;
      }
  }
}

static void cell_burgers(int Q, int ns, const double* W, const double* B, const double* D,
                         const double* consts, const double* x, const double* u, double* A) {
  const int n = 3 * ns;
  const double nu = consts[0], rdt = 1.0 / consts[1];
  double K[3][3], adet, g[20 * 3];
  geometry(x, K, &adet);
  memset(A, 0, sizeof(double) * n * n);
  for (int q = 0; q < Q; ++q) {
    phys_grad(Q, ns, q, D, K, g);
    double uq[3], gu[3][3];
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int m = 0; m < ns; ++m) s += u[c * ns + m] * B[q * ns + m];
      uq[c] = s;
      for (int d = 0; d < 3; ++d) {
        double t = 0.0;
        for (int m = 0; m < ns; ++m) t += u[c * ns + m] * g[m * 3 + d];
        gu[c][d] = t;
      }
    }
    double s = W[q] * adet;
    for (int J = 0; J < n; ++J)
      for (int Kk = 0; Kk < n; ++Kk) {
        int c = J / ns, j = J % ns, d = Kk / ns, k = Kk % ns;
        double bb = B[q * ns + j] * B[q * ns + k];
        double v = bb * (gu[c][d] + (c == d ? rdt : 0.0));
        if (c == d) {
          const double* gj = g + j * 3;
          const double* gk = g + k * 3;
          double adv = uq[0] * gk[0] + uq[1] * gk[1] + uq[2] * gk[2];
          double dif = gj[0] * gk[0] + gj[1] * gk[1] + gj[2] * gk[2];
          v += B[q * ns + j] * adv + nu * dif;
        }
        A[J * n + Kk] += v * s;
      }
  }
}

/* Element matrices for cells [0, E).  Returns 0, or -1 on a bad argument. */
int femoracle_assemble(int kind, long E, int Q, int ns, int nc, const double* W,
                       const double* B, const double* D, const double* P, const double* consts,
                       const double* coords, const double* coeffs, long ncoef, double* A) {
  int n = (kind == HELMHOLTZ) ? ns : 3 * ns;
  if (E < 0 || Q <= 0 || ns <= 0 || ns > 20) return -1;
#pragma omp parallel for schedule(static)
  for (long e = 0; e < E; ++e) {
    const double* x = coords + e * 12;
    const double* cf = coeffs + e * ncoef;
    double* Ae = A + (size_t)e * n * n;
    switch (kind) {
      case HELMHOLTZ: cell_helmholtz(Q, ns, nc, W, B, D, P, x, cf, Ae); break;
      case ELASTICITY: cell_elasticity(Q, ns, W, D, P, x, cf, Ae); break;
      case HYPERELASTICITY: cell_svk(Q, ns, W, D, P, x, cf, Ae); break;
      case BURGERS: cell_burgers(Q, ns, W, B, D, consts, x, cf, Ae); break;
      default: break;
    }
  }
  return (kind >= HELMHOLTZ && kind <= BURGERS) ? 0 : -1;
}
