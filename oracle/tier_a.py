"""Tier A oracle: the GLOBAL dense matrix A_ij = a_h(psi_j, psi_i) by brute-force quadrature.

ORACLE (test infrastructure; tiny meshes only). Follows PAPER.md term by term:
  A_ij = a_h(psi^p_j, psi^p_i)                       P:427-430 eq. linear_equation
  a_h = a^v + a^if + a^bf                            P:333-360 eq. bilinear_form_split
  jump [[v]] = v^- - v^+, {v}_w = w^- v^- + w^+ v^+  P:376-389
  w^± = delta^∓/(delta^- + delta^+), delta = nu^T K nu
  gamma_F = alpha p (p+d-1) <d^-,d^+>|F|/min|T|  or  d^-|F|/|T^-|
  upwind Phi(u^-, u^+, b_nu)
  l_h(v)                                             P:361-371 eq. rhs
Every 3D basis function is evaluated directly at every quadrature point as the
tensor product of 1D Lagrange polynomials (no sum factorisation); K may be a
full 3x3 matrix per cell; b may vary per cell (face b_nu = nu . (b^- + b^+)/2,
SURVEY §8(c) reading #8). Quadrature: m_o = p+3 Gauss points per direction
(exact for all integrands here, reading #4).
"""
from __future__ import annotations

import numpy as np

from synth.problem import DIRICHLET, NEUMANN, Problem
from .basis import (face_weights, gauss_rule, harmonic_average, lagrange_derivs,
                    lagrange_values, lobatto_nodes)


def _K_full(P: Problem, K_full):
    if K_full is not None:
        return np.asarray(K_full, dtype=np.float64)
    K3 = P.K3()
    return np.einsum("na,ab->nab", K3, np.eye(3))


def _b_cells(P: Problem, b_cells):
    if b_cells is not None:
        return np.asarray(b_cells, dtype=np.float64)
    return P.b3()


class TierA:
    def __init__(self, P: Problem, K_full=None, b_cells=None, m_o=None):
        self.P = P
        self.n = P.p + 1
        self.nd = self.n ** 3
        self.m = (P.p + 3) if m_o is None else m_o
        self.nodes = lobatto_nodes(P.p)
        self.xq, self.wq = gauss_rule(self.m)
        self.K = _K_full(P, K_full)
        self.b = _b_cells(P, b_cells)
        self.cvec = P.c_cells()
        self.h = np.array(P.h)

    # ---- geometry -------------------------------------------------------
    def cell_index(self, cx, cy, cz):
        P = self.P
        return cx + P.nx * (cy + P.ny * cz)

    def cell_coords(self, c):
        P = self.P
        return c % P.nx, (c // P.nx) % P.ny, c // (P.nx * P.ny)

    def origin(self, c):
        return np.array(self.cell_coords(c), dtype=np.float64) * self.h

    # ---- basis evaluation at arbitrary reference points -------------------
    def eval_basis(self, Xhat):
        """Values [Q, nd] and physical gradients [Q, nd, 3] of all psi_I at reference
        points Xhat [Q, 3]; I = i + n j + n^2 k (x fastest)."""
        n = self.n
        Vx, Vy, Vz = (lagrange_values(self.nodes, Xhat[:, a]) for a in range(3))
        Gx, Gy, Gz = (lagrange_derivs(self.nodes, Xhat[:, a]) for a in range(3))
        val = np.einsum("qk,qj,qi->qkji", Vz, Vy, Vx).reshape(-1, n ** 3)
        gx = np.einsum("qk,qj,qi->qkji", Vz, Vy, Gx).reshape(-1, n ** 3) / self.h[0]
        gy = np.einsum("qk,qj,qi->qkji", Vz, Gy, Vx).reshape(-1, n ** 3) / self.h[1]
        gz = np.einsum("qk,qj,qi->qkji", Gz, Vy, Vx).reshape(-1, n ** 3) / self.h[2]
        return val, np.stack([gx, gy, gz], axis=2)

    def volume_points(self):
        x = self.xq
        X = np.stack(np.meshgrid(x, x, x, indexing="ij"), axis=-1).reshape(-1, 3)  # any order
        w = np.einsum("a,b,c->abc", self.wq, self.wq, self.wq).reshape(-1)
        return X, w

    def face_points(self, axis, coord):
        """Reference points on the face x_axis = coord of the unit cube, and 2D weights."""
        x = self.xq
        t1, t2 = [a for a in range(3) if a != axis]
        A, B = np.meshgrid(x, x, indexing="ij")
        X = np.zeros((A.size, 3))
        X[:, t1] = A.reshape(-1)
        X[:, t2] = B.reshape(-1)
        X[:, axis] = coord
        w = np.einsum("a,b->ab", self.wq, self.wq).reshape(-1)
        return X, w

    def measure(self):
        hx, hy, hz = self.h
        return hx * hy * hz, (hy * hz, hx * hz, hx * hy)

    # ---- a^v -------------------------------------------------------------
    def volume_block(self, c):
        """(A^v_{T,T})_{IJ} = a^v(psi_J, psi_I) = sum_q w_q |T| [(K grad psi_J - b psi_J).grad psi_I
        + c psi_J psi_I]."""
        X, w = self.volume_points()
        val, grad = self.eval_basis(X)
        vol, _ = self.measure()
        K, b, cc = self.K[c], self.b[c], self.cvec[c]
        Kg = np.einsum("ab,qJb->qJa", K, grad)                   # K grad psi_J
        flux = Kg - b[None, None, :] * val[:, :, None]           # K grad u - b u
        Aloc = np.einsum("q,qJa,qIa->IJ", w * vol, flux, grad)
        Aloc += cc * np.einsum("q,qJ,qI->IJ", w * vol, val, val)
        return Aloc

    # ---- a^if: the four (T', T'') contributions of one interior face ------
    def interior_face_blocks(self, cl, cu, axis, flip=False):
        """Blocks {(test_cell, trial_cell): matrix} of a^if restricted to the face between the
        lower cell cl and the upper cell cu. flip=True orients nu = -e_axis, so
        the '-' side is the upper cell (the result must not change; SURVEY §8(c) reading #5)."""
        P = self.P
        _, areas = self.measure()
        vol, _ = self.measure()
        area = areas[axis]
        Xl, w = self.face_points(axis, 1.0)   # face seen from the lower cell
        Xu, _ = self.face_points(axis, 0.0)   # same physical points seen from the upper cell
        vl, gl = self.eval_basis(Xl)
        vu, gu = self.eval_basis(Xu)
        e = np.zeros(3)
        e[axis] = 1.0
        if not flip:
            nu = e
            side = {"-": (cl, vl, gl), "+": (cu, vu, gu)}
        else:
            nu = -e
            side = {"-": (cu, vu, gu), "+": (cl, vl, gl)}
        cm, cp = side["-"][0], side["+"][0]
        dm = nu @ self.K[cm] @ nu
        dp = nu @ self.K[cp] @ nu
        wm, wp = face_weights(dm, dp)
        omega = {"-": wm, "+": wp}
        gamma = P.alpha * P.p * (P.p + 2) * harmonic_average(dm, dp) * area / vol
        bnu = nu @ (0.5 * (self.b[cm] + self.b[cp]))
        sign = {"-": 1.0, "+": -1.0}
        data = {}
        for s in ("-", "+"):
            cs, v, g = side[s]
            jump = sign[s] * v                                     # [[psi]] of a side-s function
            avg = omega[s] * np.einsum("a,ab,qIb->qI", nu, self.K[cs], g)  # nu.{K grad psi}_w
            if (bnu >= 0 and s == "-") or (bnu < 0 and s == "+"):
                phi = bnu * v                                      # Phi(psi^-, psi^+, b_nu)
            else:
                phi = np.zeros_like(v)
            data[s] = (cs, jump, avg, phi)
        blocks = {}
        wt = w * area
        for st in ("-", "+"):          # test side
            ct, jt, at, _ = data[st]
            for sr in ("-", "+"):      # trial side
                cr, jr, ar, phr = data[sr]
                M = (np.einsum("q,qJ,qI->IJ", wt, phr, jt)
                     - np.einsum("q,qJ,qI->IJ", wt, ar, jt)
                     - np.einsum("q,qI,qJ->IJ", wt, at, jr)
                     + gamma * np.einsum("q,qJ,qI->IJ", wt, jr, jt))
                blocks[(ct, cr)] = blocks.get((ct, cr), 0.0) + M
        return blocks

    # ---- a^bf ------------------------------------------------------------
    def boundary_face_block(self, c, axis, hi):
        """Dirichlet face term a^bf(psi_J, psi_I); Neumann faces give 0."""
        P = self.P
        kind = P.bc[2 * axis + (1 if hi else 0)]
        if kind == NEUMANN:
            return np.zeros((self.nd, self.nd))
        vol, areas = self.measure()
        area = areas[axis]
        X, w = self.face_points(axis, 1.0 if hi else 0.0)
        v, g = self.eval_basis(X)
        nu = np.zeros(3)
        nu[axis] = 1.0 if hi else -1.0
        K = self.K[c]
        delta = nu @ K @ nu
        gamma = P.alpha * P.p * (P.p + 2) * delta * area / vol
        bnu = nu @ self.b[c]
        phi = bnu * v if bnu >= 0 else np.zeros_like(v)      # Phi(u, 0, b_nu)
        fl = np.einsum("a,ab,qIb->qI", nu, K, g)               # nu . K grad psi
        wt = w * area
        return (np.einsum("q,qJ,qI->IJ", wt, phi, v)
                - np.einsum("q,qJ,qI->IJ", wt, fl, v)
                - np.einsum("q,qI,qJ->IJ", wt, fl, v)
                + gamma * np.einsum("q,qJ,qI->IJ", wt, v, v))

    # ---- global assembly ---------------------------------------------------
    def assemble(self, flip=False):
        P = self.P
        nd, N = self.nd, P.n_cells
        A = np.zeros((N * nd, N * nd))

        def add(ct, cr, M):
            A[ct * nd:(ct + 1) * nd, cr * nd:(cr + 1) * nd] += M

        for c in range(N):
            add(c, c, self.volume_block(c))
        dims = (P.nx, P.ny, P.nz)
        for c in range(N):
            co = list(self.cell_coords(c))
            for axis in range(3):
                if co[axis] + 1 < dims[axis]:
                    cu_co = list(co)
                    cu_co[axis] += 1
                    cu = self.cell_index(*cu_co)
                    for (ct, cr), M in self.interior_face_blocks(c, cu, axis, flip).items():
                        add(ct, cr, M)
                if co[axis] == 0:
                    add(c, c, self.boundary_face_block(c, axis, hi=False))
                if co[axis] == dims[axis] - 1:
                    add(c, c, self.boundary_face_block(c, axis, hi=True))
        return A

    # ---- right-hand side l_h -------------------------------------------------
    def rhs(self, f, g, j):
        """l_h(psi_I). f(X) volume source, g(X) Dirichlet data, j(X, nu) Neumann
        flux data; X physical points [Q, 3]."""
        P = self.P
        nd, N = self.nd, P.n_cells
        out = np.zeros(N * nd)
        vol, areas = self.measure()
        Xv, wv = self.volume_points()
        val, _ = self.eval_basis(Xv)
        dims = (P.nx, P.ny, P.nz)
        for c in range(N):
            o = self.origin(c)
            out[c * nd:(c + 1) * nd] += np.einsum("q,q,qI->I", wv * vol, f(o + Xv * self.h), val)
            co = self.cell_coords(c)
            for axis in range(3):
                for hi in (False, True):
                    if (not hi and co[axis] != 0) or (hi and co[axis] != dims[axis] - 1):
                        continue
                    kind = P.bc[2 * axis + (1 if hi else 0)]
                    X, w = self.face_points(axis, 1.0 if hi else 0.0)
                    v, gr = self.eval_basis(X)
                    Xp = o + X * self.h
                    nu = np.zeros(3)
                    nu[axis] = 1.0 if hi else -1.0
                    wt = w * areas[axis]
                    if kind == NEUMANN:
                        out[c * nd:(c + 1) * nd] -= np.einsum("q,q,qI->I", wt, j(Xp, nu), v)
                        continue
                    K = self.K[c]
                    delta = nu @ K @ nu
                    gamma = P.alpha * P.p * (P.p + 2) * delta * areas[axis] / vol
                    bnu = nu @ self.b[c]
                    gv = g(Xp)
                    phi = bnu * gv if bnu < 0 else np.zeros_like(gv)    # Phi(0, g, b_nu)
                    fl = np.einsum("a,ab,qIb->qI", nu, K, gr)
                    out[c * nd:(c + 1) * nd] -= (np.einsum("q,q,qI->I", wt, phi, v)
                                                 + np.einsum("q,qI,q->I", wt, fl, gv)
                                                 - gamma * np.einsum("q,q,qI->I", wt, gv, v))
        return out

    def interpolate(self, ufun):
        """Nodal interpolant: coefficient of psi_I = u(zeta_I) (nodal basis)."""
        P = self.P
        n = self.n
        z = self.nodes
        Xhat = np.zeros((n ** 3, 3))      # node I = i + n j + n^2 k sits at (z_i, z_j, z_k)
        for k in range(n):
            for jj in range(n):
                for i in range(n):
                    Xhat[i + n * jj + n * n * k] = (z[i], z[jj], z[k])
        out = np.zeros(P.n_cells * self.nd)
        for c in range(P.n_cells):
            out[c * self.nd:(c + 1) * self.nd] = ufun(self.origin(c) + Xhat * self.h)
        return out
