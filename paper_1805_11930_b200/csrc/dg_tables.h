// 1D tables of the nodal Gauss-Lobatto basis and the Gauss rule on [0,1] (host side).
//
// Paper: tensor-product Lagrange basis on Gauss-Lobatto nodes (§2.1),
// tensor Gauss rule with m = n = p+1 points (§3.1, "typically m=n=p+1").
// Built here from scratch (Newton iterations on Legendre polynomials); nothing is
// shared with oracle/.
#pragma once
#include <cstdint>

namespace dg {

constexpr int kMaxN = 8;  // p <= 7

struct Tables1D {
  int n;                       // p + 1 (nodes == quadrature points)
  double z[kMaxN];             // GL nodes
  double xq[kMaxN], wq[kMaxN]; // Gauss points / weights
  double A[kMaxN * kMaxN];     // A[q*n+j] = theta_j(xi_q)       (P:850 A^(k))
  double G[kMaxN * kMaxN];     // G[q*n+j] = theta_j'(xi_q)
  double D[kMaxN * kMaxN];     // D[q*n+r] = l_r'(xi_q): collocation derivative at Gauss points (D A = G)
  double M[kMaxN * kMaxN];     // Mhat = A^T W A (exact 1D mass, also the face mass factor)
  double d0[kMaxN], d1[kMaxN]; // theta_j'(0), theta_j'(1)
  double Sdiag[kMaxN];         // diag of Shat = G^T W G
  double Cdiag[kMaxN];         // diag of Chat = G^T W A (test derivative)
  double Mdiag[kMaxN];
  // Gauss-point Lagrange polynomials l_q evaluated at the cell ends: E0[q] = l_q(0), E1[q] = l_q(1),
  // F0[q] = l_q'(0), F1[q] = l_q'(1). Trace / normal derivative of a polynomial from its Gauss
  // values U: u(0) = E0.U, u'(0) = F0.U; and A^T E0 = e0, A^T F0 = d0 (used to inject face terms).
  double E0[kMaxN], E1[kMaxN], F0[kMaxN], F1[kMaxN];
};

// Fills t for degree p (1..7). Returns false on invalid p.
bool build_tables(int p, Tables1D* t);

}  // namespace dg
