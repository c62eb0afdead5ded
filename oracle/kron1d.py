"""1D global SIPG operators and the exact Kronecker-sum reduction of the 3D operator.

ORACLE (test infrastructure). For K = kappa I, b = 0, c = 0 and all-Dirichlet
boundaries on a uniform box, A equals, in the permuted tensor ordering
(X = cx n + i, Y = cy n + j, Z = cz n + k),
    A = kappa (A1_z . M1_y . M1_x + M1_z . A1_y . M1_x + M1_z . M1_y . A1_x)
with A1 the 1D global interior-penalty operator with penalty alpha p(p+2)/h and
weights 1/2, and M1 the 1D global (block-diagonal) mass matrix. The 1D operators
are assembled here by brute-force 1D quadrature of the 1D form
    int u'v' - sum_F ({u'} [v] + {v'} [u]) + gamma [u][v]
so this module is an independent route to A. For separable u = ux . uy . uz the
exact Au costs O(N^(1/3)) per factor: it pins dg_apply at full C1/C2 size.
"""
from __future__ import annotations

import numpy as np

from .basis import gauss_rule, lagrange_derivs, lagrange_values, lobatto_nodes


def sipg_1d(ncell: int, L: float, p: int, alpha: float):
    """(A1, M1): 1D global SIPG stiffness (Dirichlet at both ends) and mass, size ncell*(p+1)."""
    n = p + 1
    h = L / ncell
    z = lobatto_nodes(p)
    xq, wq = gauss_rule(p + 3)
    V = lagrange_values(z, xq)
    G = lagrange_derivs(z, xq) / h
    v0 = lagrange_values(z, [0.0])[0]
    v1 = lagrange_values(z, [1.0])[0]
    g0 = lagrange_derivs(z, [0.0])[0] / h
    g1 = lagrange_derivs(z, [1.0])[0] / h
    N = ncell * n
    A = np.zeros((N, N))
    M = np.zeros((N, N))
    gamma = alpha * p * (p + 2) / h
    for c in range(ncell):
        s = slice(c * n, (c + 1) * n)
        A[s, s] += h * np.einsum("q,qi,qj->ij", wq, G, G)
        M[s, s] += h * np.einsum("q,qi,qj->ij", wq, V, V)
    # interior points x_F between cell c (left, '-') and c+1 (right, '+'), nu = +1
    for c in range(ncell - 1):
        sides = {"-": (c, v1, g1), "+": (c + 1, v0, g0)}
        sgn = {"-": 1.0, "+": -1.0}
        for st in "-+":
            ct, vt, gt = sides[st]
            for sr in "-+":
                cr, vr, gr = sides[sr]
                blk = (-np.outer(sgn[st] * vt, 0.5 * gr)       # -{u'} [v]
                       - np.outer(0.5 * gt, sgn[sr] * vr)      # -{v'} [u]
                       + gamma * np.outer(sgn[st] * vt, sgn[sr] * vr))
                A[ct * n:(ct + 1) * n, cr * n:(cr + 1) * n] += blk
    # Dirichlet ends: nu = -1 at x=0, +1 at x=L
    for c, v, g, nu in ((0, v0, g0, -1.0), (ncell - 1, v1, g1, 1.0)):
        s = slice(c * n, (c + 1) * n)
        A[s, s] += (-np.outer(v, nu * g) - np.outer(nu * g, v) + gamma * np.outer(v, v))
    return A, M


def separable_apply(P, ux, uy, uz, kappa=1.0):
    """Exact A (ux . uy . uz) for the K = kappa I, b = c = 0, all-Dirichlet problem,
    returned in the cell-major DoF layout (c = cx + nx (cy + ny cz), I = i + n j + n^2 k)."""
    Ax, Mx = sipg_1d(P.nx, P.Lx, P.p, P.alpha)
    Ay, My = sipg_1d(P.ny, P.Ly, P.p, P.alpha)
    Az, Mz = sipg_1d(P.nz, P.Lz, P.p, P.alpha)
    terms = [(Ax @ ux, My @ uy, Mz @ uz), (Mx @ ux, Ay @ uy, Mz @ uz), (Mx @ ux, My @ uy, Az @ uz)]
    return kappa * sum(to_cell_major(P, a, b, c) for a, b, c in terms)


def to_cell_major(P, fx, fy, fz):
    """Tensor product fx[X] fy[Y] fz[Z] in the cell-major layout."""
    n = P.p + 1
    tx = fx.reshape(P.nx, n)      # [cx, i]
    ty = fy.reshape(P.ny, n)
    tz = fz.reshape(P.nz, n)
    # out[cz, cy, cx, k, j, i]
    out = np.einsum("ck,bj,ai->cbakji", tz, ty, tx)
    return out.reshape(-1)
