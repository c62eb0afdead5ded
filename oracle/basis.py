"""1D nodal Gauss-Lobatto Lagrange basis and Gauss-Legendre quadrature on [0, 1].

ORACLE (test infrastructure). Paper: "tensor-product of one-dimensional
Gauss-Lobatto basis functions (i.e. Lagrange polynomials with nodes at the
Gauss-Lobatto points)" and nodal psi_i(zeta_j) = delta_ij (§2.1);
tensor Gauss rule with m points per direction (§3.1).

Library primitives used as steps: numpy.polynomial.legendre (roots of P_p',
Gauss-Legendre rule). Lagrange values/derivatives are the product formula.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as L


def lobatto_nodes(p: int) -> np.ndarray:
    """GL nodes on [0,1]: {0, 1} and the roots of P_p' mapped from [-1,1]."""
    if p < 1:
        raise ValueError("p >= 1")
    inner = np.array([]) if p == 1 else np.sort(L.Legendre.basis(p).deriv().roots().real)
    x = np.concatenate([[-1.0], inner, [1.0]])
    return 0.5 * (x + 1.0)


def gauss_rule(m: int):
    """m-point Gauss-Legendre rule on [0,1]: (points, weights)."""
    x, w = L.leggauss(m)
    return 0.5 * (x + 1.0), 0.5 * w


def lagrange_values(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """V[q, i] = theta_i(x_q) = prod_{j != i} (x_q - z_j) / (z_i - z_j)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    V = np.ones((len(x), n))
    for i in range(n):
        for j in range(n):
            if j != i:
                V[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return V


def lagrange_derivs(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """G[q, i] = theta_i'(x_q) by the product rule:
    sum_{l != i} 1/(z_i - z_l) * prod_{j != i, l} (x_q - z_j)/(z_i - z_j)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    G = np.zeros((len(x), n))
    for i in range(n):
        for l in range(n):
            if l == i:
                continue
            term = np.full(len(x), 1.0 / (nodes[i] - nodes[l]))
            for j in range(n):
                if j != i and j != l:
                    term *= (x - nodes[j]) / (nodes[i] - nodes[j])
            G[:, i] += term
    return G


def harmonic_average(a: float, b: float) -> float:
    """<a,b> = 2ab/(a+b); 0 when a+b = 0 (SURVEY §8(c) reading #7)."""
    return 0.0 if a + b == 0.0 else 2.0 * a * b / (a + b)


def face_weights(dm: float, dp: float):
    """omega^± = delta^∓ / (delta^- + delta^+); 1/2 each if degenerate."""
    s = dm + dp
    if s == 0.0:
        return 0.5, 0.5
    return dp / s, dm / s


def upwind(um, up, bnu):
    """Phi(u^-, u^+, b_nu) = b_nu u^- if b_nu >= 0 else b_nu u^+ (P:407-414)."""
    return bnu * um if bnu >= 0 else bnu * up
