// 1D GL basis / Gauss rule tables (see dg_tables.h).
#include "dg_tables.h"

#include <cmath>

namespace dg {
namespace {

// Legendre P_k(x) and its derivative on [-1,1] by the three-term recurrence.
void legendre(int k, double x, double* P, double* dP) {
  double p0 = 1.0, p1 = x;
  if (k == 0) { *P = 1.0; *dP = 0.0; return; }
  for (int j = 2; j <= k; ++j) {
    double p2 = ((2.0 * j - 1.0) * x * p1 - (j - 1.0) * p0) / j;
    p0 = p1;
    p1 = p2;
  }
  *P = p1;
  *dP = (std::fabs(x) < 1.0) ? k * (x * p1 - p0) / (x * x - 1.0) : 0.5 * k * (k + 1) * std::pow(x, k + 1);
}

// Gauss-Legendre rule with m points on [-1,1] (Newton on P_m from Chebyshev guesses).
void gauss_pm1(int m, double* x, double* w) {
  for (int i = 0; i < m; ++i) {
    double r = -std::cos(M_PI * (i + 0.75) / (m + 0.5));
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre(m, r, &P, &dP);
      double dr = P / dP;
      r -= dr;
      if (std::fabs(dr) < 1e-16) break;
    }
    double P, dP;
    legendre(m, r, &P, &dP);
    x[i] = r;
    w[i] = 2.0 / ((1.0 - r * r) * dP * dP);
  }
}

// Interior GL nodes: roots of P_p' via Newton, with P_p'' from the Legendre ODE
// (1-x^2) P'' = 2x P' - p(p+1) P.
void lobatto_pm1(int p, double* z) {
  int n = p + 1;
  z[0] = -1.0;
  z[n - 1] = 1.0;
  for (int i = 1; i < n - 1; ++i) {
    double r = -std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre(p, r, &P, &dP);
      double d2P = (2.0 * r * dP - p * (p + 1.0) * P) / (1.0 - r * r);
      double dr = dP / d2P;
      r -= dr;
      if (std::fabs(dr) < 1e-16) break;
    }
    z[i] = r;
  }
}

double lagrange(const double* nodes, int n, int i, double x) {
  double v = 1.0;
  for (int j = 0; j < n; ++j)
    if (j != i) v *= (x - nodes[j]) / (nodes[i] - nodes[j]);
  return v;
}

double lagrange_d(const double* nodes, int n, int i, double x) {
  double s = 0.0;
  for (int l = 0; l < n; ++l) {
    if (l == i) continue;
    double t = 1.0 / (nodes[i] - nodes[l]);
    for (int j = 0; j < n; ++j)
      if (j != i && j != l) t *= (x - nodes[j]) / (nodes[i] - nodes[j]);
    s += t;
  }
  return s;
}

}  // namespace

bool build_tables(int p, Tables1D* t) {
  if (p < 1 || p > kMaxN - 1) return false;
  const int n = p + 1;
  *t = Tables1D{};
  t->n = n;
  double zz[kMaxN], xx[kMaxN], ww[kMaxN];
  lobatto_pm1(p, zz);
  gauss_pm1(n, xx, ww);
  for (int i = 0; i < n; ++i) {
    t->z[i] = 0.5 * (zz[i] + 1.0);
    t->xq[i] = 0.5 * (xx[i] + 1.0);
    t->wq[i] = 0.5 * ww[i];
  }
  t->z[0] = 0.0;
  t->z[n - 1] = 1.0;
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j) {
      t->A[q * n + j] = lagrange(t->z, n, j, t->xq[q]);
      t->G[q * n + j] = lagrange_d(t->z, n, j, t->xq[q]);
      t->D[q * n + j] = lagrange_d(t->xq, n, j, t->xq[q]);
    }
  for (int i = 0; i < n; ++i) {
    t->d0[i] = lagrange_d(t->z, n, i, 0.0);
    t->d1[i] = lagrange_d(t->z, n, i, 1.0);
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int q = 0; q < n; ++q) s += t->wq[q] * t->A[q * n + i] * t->A[q * n + j];
      t->M[i * n + j] = s;
    }
    double sd = 0.0, cd = 0.0;
    for (int q = 0; q < n; ++q) {
      sd += t->wq[q] * t->G[q * n + i] * t->G[q * n + i];
      cd += t->wq[q] * t->G[q * n + i] * t->A[q * n + i];
    }
    t->Sdiag[i] = sd;
    t->Cdiag[i] = cd;
    t->Mdiag[i] = t->M[i * n + i];
    t->E0[i] = lagrange(t->xq, n, i, 0.0);
    t->E1[i] = lagrange(t->xq, n, i, 1.0);
    t->F0[i] = lagrange_d(t->xq, n, i, 0.0);
    t->F1[i] = lagrange_d(t->xq, n, i, 1.0);
  }
  return true;
}

}  // namespace dg
