"""Tier B oracle: per-cell dense blocks from 1D brute-force quadrature + Kronecker products.

ORACLE (test infrastructure; timed as the CPU baseline). For per-cell constant,
diagonal K, per-cell constant b, c on a uniform axis-aligned box, every block of
A (eq. block_ls) is a Kronecker product of 1D matrices. Derivation
(DESIGN.md §"Oracle", restating SURVEY.md §8(c) step 3 from P:343-357 with
nu = n_T and P:376-389 for the orientation):
  1D on [0,1], m_o = p+3 Gauss points:  Mh_ij = int th_i th_j,  Sh_ij = int th_i' th_j',
  Ch_ij = int th_i' th_j (test derivative);  e0, e1 unit vectors at the end nodes,
  d0 = th'(0), d1 = th'(1).  Physical: M = h Mh, S = Sh / h, C = Ch.
  DoF I = i + n j + n^2 k  ->  operators are kron(Z, kron(Y, X)).
  Volume:  Kx Mz.My.Sx + Ky Mz.Sy.Mx + Kz Sz.My.Mx - bx Mz.My.Cx - by Mz.Cy.Mx - bz Cz.My.Mx
           + c Mz.My.Mx                                                  (a^v)
  x+ face self:  F_x . [max(bn,0) e1e1' - wT KTx (e1 d1' + d1 e1')/hx + g e1e1']
  x- face self:  F_x . [max(-bn,0) e0e0' + wT KTx (e0 d0' + d0 e0')/hx + g e0e0']
  x+ neighbour:  F_x . [min(bn,0) e1e0' - wN KNx e1 d0'/hx + wT KTx d1 e0'/hx - g e1e0']
  x- neighbour:  F_x . [min(-bn,0) e0e1' + wN KNx e0 d1'/hx - wT KTx d0 e1'/hx - g e0e1']
  F_x = Mz.My (tangential face mass); same pattern for y, z.   (a^if)
  Dirichlet face: self form with w = 1, g = alpha p(p+2) K/h; Neumann: 0.   (a^bf)
  interior g = alpha p(p+2) <dT, dN> / h_axis  (|F|/min|T| = 1/h_axis on the uniform box).
The block-Jacobi sweep (Alg. 2) uses exact local solves by LU with
partial pivoting (numpy.linalg.solve) of D_T = A_{T,T}.
"""
from __future__ import annotations

import numpy as np

from synth.problem import DIRICHLET, NEUMANN, Problem
from .basis import (face_weights, gauss_rule, harmonic_average, lagrange_derivs,
                    lagrange_values, lobatto_nodes)


def kron3(Z, Y, X):
    return np.kron(Z, np.kron(Y, X))


class TierB:
    def __init__(self, P: Problem, m_o=None, b_cells=None):
        self.P = P
        self.n = n = P.p + 1
        self.nd = n ** 3
        m = (P.p + 3) if m_o is None else m_o
        z = lobatto_nodes(P.p)
        xq, wq = gauss_rule(m)
        V = lagrange_values(z, xq)
        G = lagrange_derivs(z, xq)
        self.Mh = np.einsum("q,qi,qj->ij", wq, V, V)
        self.Sh = np.einsum("q,qi,qj->ij", wq, G, G)
        self.Ch = np.einsum("q,qi,qj->ij", wq, G, V)      # test derivative i, trial j
        self.e0 = lagrange_values(z, [0.0])[0]
        self.e1 = lagrange_values(z, [1.0])[0]
        self.d0 = lagrange_derivs(z, [0.0])[0]
        self.d1 = lagrange_derivs(z, [1.0])[0]
        self.h = np.array(P.h)
        self.K = P.K3()
        self.b = P.b3() if b_cells is None else np.asarray(b_cells, dtype=np.float64)
        self.c = P.c_cells()
        self.dims = (P.nx, P.ny, P.nz)

    # ---- mesh -----------------------------------------------------------
    def coords(self, c):
        P = self.P
        return [c % P.nx, (c // P.nx) % P.ny, c // (P.nx * P.ny)]

    def index(self, co):
        P = self.P
        return co[0] + P.nx * (co[1] + P.ny * co[2])

    def neighbour(self, c, axis, hi):
        co = self.coords(c)
        co[axis] += 1 if hi else -1
        if co[axis] < 0 or co[axis] >= self.dims[axis]:
            return None
        return self.index(co)

    # ---- 1D physical matrices -------------------------------------------
    def M1(self, a):
        return self.h[a] * self.Mh

    def embed(self, axis, B):
        """kron with the 1D matrix B in direction `axis` and physical masses elsewhere."""
        ops = [self.M1(0), self.M1(1), self.M1(2)]
        ops[axis] = B
        return kron3(ops[2], ops[1], ops[0])

    # ---- blocks -----------------------------------------------------------
    def volume_block(self, c):
        K, b, cc = self.K[c], self.b[c], self.c[c]
        A = np.zeros((self.nd, self.nd))
        for a in range(3):
            A += K[a] * self.embed(a, self.Sh / self.h[a])
            A -= b[a] * self.embed(a, self.Ch)
        A += cc * kron3(self.M1(2), self.M1(1), self.M1(0))
        return A

    def face_params(self, c, axis, hi):
        """(kind, omega_T, omega_N, gamma, b_nu, K_Tk, K_Nk, nbr) of the face of c on side hi;
        b_nu = (face b) . e_axis for interior faces, (b_T . outward nu) for boundary faces."""
        P = self.P
        nb = self.neighbour(c, axis, hi)
        KT = self.K[c, axis]
        pp = P.alpha * P.p * (P.p + 2)
        if nb is None:
            kind = P.bc[2 * axis + (1 if hi else 0)]
            bnu = self.b[c, axis] * (1.0 if hi else -1.0)
            return kind, 1.0, 0.0, pp * KT / self.h[axis], bnu, KT, 0.0, None
        KN = self.K[nb, axis]
        wT, wN = face_weights(KT, KN)  # omega_T = delta_N/(delta_T + delta_N)
        gamma = pp * harmonic_average(KT, KN) / self.h[axis]
        bnu = 0.5 * (self.b[c, axis] + self.b[nb, axis])
        return "interior", wT, wN, gamma, bnu, KT, KN, nb

    def self_face_1d(self, c, axis, hi):
        kind, wT, wN, g, bn, KT, KN, nb = self.face_params(c, axis, hi)
        hk = self.h[axis]
        e0, e1, d0, d1 = self.e0, self.e1, self.d0, self.d1
        if kind == NEUMANN:
            return np.zeros((self.n, self.n))
        o = np.outer
        if kind == DIRICHLET:
            # outward normal: bn already b . nu
            if hi:
                return max(bn, 0.0) * o(e1, e1) - KT * (o(e1, d1) + o(d1, e1)) / hk + g * o(e1, e1)
            return max(bn, 0.0) * o(e0, e0) + KT * (o(e0, d0) + o(d0, e0)) / hk + g * o(e0, e0)
        if hi:
            return max(bn, 0.0) * o(e1, e1) - wT * KT * (o(e1, d1) + o(d1, e1)) / hk + g * o(e1, e1)
        return max(-bn, 0.0) * o(e0, e0) + wT * KT * (o(e0, d0) + o(d0, e0)) / hk + g * o(e0, e0)

    def nbr_face_1d(self, c, axis, hi):
        kind, wT, wN, g, bn, KT, KN, nb = self.face_params(c, axis, hi)
        if nb is None:
            return None, None
        hk = self.h[axis]
        e0, e1, d0, d1 = self.e0, self.e1, self.d0, self.d1
        o = np.outer
        if hi:
            B = min(bn, 0.0) * o(e1, e0) - wN * KN * o(e1, d0) / hk + wT * KT * o(d1, e0) / hk - g * o(e1, e0)
        else:
            B = min(-bn, 0.0) * o(e0, e1) + wN * KN * o(e0, d1) / hk - wT * KT * o(d0, e1) / hk - g * o(e0, e1)
        return nb, B

    def diag_block(self, c):
        """D_T = A^v_{T,T} + sum of self-face terms (P:893-903 eq. block_diag_apply)."""
        D = self.volume_block(c)
        for axis in range(3):
            for hi in (False, True):
                D += self.embed(axis, self.self_face_1d(c, axis, hi))
        return D

    def nbr_blocks(self, c):
        """[(N, A_{T,N})] for the face neighbours of c (minimal stencil)."""
        out = []
        for axis in range(3):
            for hi in (False, True):
                nb, B = self.nbr_face_1d(c, axis, hi)
                if nb is not None:
                    out.append((nb, self.embed(axis, B)))
        return out

    # ---- operator application ----------------------------------------------
    def apply_cells(self, u, cells):
        """(A u)_T for T in cells, as dense nd x nd block matvecs (returns [len(cells), nd])."""
        nd = self.nd
        U = np.asarray(u).reshape(-1, nd)
        out = np.zeros((len(cells), nd))
        for r, c in enumerate(cells):
            out[r] = self.diag_block(c) @ U[c]
            for nb, B in self.nbr_blocks(c):
                out[r] += B @ U[nb]
        return out

    def apply(self, u):
        return self.apply_cells(u, range(self.P.n_cells)).reshape(-1)

    def apply_parts_cells(self, u, cells, mask):
        """Selected parts of (A u)_T: mask 1 = a^v, 2 = a^if (self + neighbour), 4 = a^bf."""
        nd = self.nd
        U = np.asarray(u).reshape(-1, nd)
        out = np.zeros((len(cells), nd))
        for r, c in enumerate(cells):
            if mask & 1:
                out[r] += self.volume_block(c) @ U[c]
            for axis in range(3):
                for hi in (False, True):
                    interior = self.neighbour(c, axis, hi) is not None
                    if (interior and mask & 2) or (not interior and mask & 4):
                        out[r] += self.embed(axis, self.self_face_1d(c, axis, hi)) @ U[c]
                    if interior and mask & 2:
                        nb, B = self.nbr_face_1d(c, axis, hi)
                        out[r] += self.embed(axis, B) @ U[nb]
        return out

    def volume_apply(self, u):
        """A^v u for every cell at once: volume_block's sum of coefficient-weighted Kronecker
        operators, applied to all cells (rows of U) by linearity (large meshes)."""
        U = np.asarray(u).reshape(-1, self.nd)
        out = np.zeros_like(U)
        for a in range(3):
            out += self.K[:, a:a + 1] * (U @ self.embed(a, self.Sh / self.h[a]).T)
            out -= self.b[:, a:a + 1] * (U @ self.embed(a, self.Ch).T)
        out += self.c[:, None] * (U @ kron3(self.M1(2), self.M1(1), self.M1(0)).T)
        return out.reshape(-1)

    def block_diag_apply(self, u, cells=None):
        cells = range(self.P.n_cells) if cells is None else cells
        U = np.asarray(u).reshape(-1, self.nd)
        return np.stack([self.diag_block(c) @ U[c] for c in cells])

    def assemble(self):
        nd, N = self.nd, self.P.n_cells
        A = np.zeros((N * nd, N * nd))
        for c in range(N):
            A[c * nd:(c + 1) * nd, c * nd:(c + 1) * nd] = self.diag_block(c)
            for nb, B in self.nbr_blocks(c):
                A[c * nd:(c + 1) * nd, nb * nd:(nb + 1) * nd] += B
        return A

    # ---- local solves and the block-Jacobi sweep (Alg. 2) --------------------
    def local_solve(self, d, cells=None):
        """delta_T = D_T^{-1} d_T by LU with partial pivoting (exact block solve)."""
        cells = range(self.P.n_cells) if cells is None else list(cells)
        Dv = np.asarray(d).reshape(-1, self.nd)
        rows = Dv if Dv.shape[0] == len(cells) else Dv[list(cells)]
        return np.stack([np.linalg.solve(self.diag_block(c), rows[r]) for r, c in enumerate(cells)])

    def sweep_cells(self, u, f, omega, cells):
        """Alg. 2 lines 2-4 restricted to `cells`: d = f - A u; D_T du_T = d_T; u_T + omega du_T."""
        nd = self.nd
        U = np.asarray(u).reshape(-1, nd)
        F = np.asarray(f).reshape(-1, nd)
        cells = list(cells)
        Au = self.apply_cells(u, cells)
        out = np.zeros((len(cells), nd))
        for r, c in enumerate(cells):
            d = F[c] - Au[r]
            out[r] = U[c] + omega * np.linalg.solve(self.diag_block(c), d)
        return out

    def sweep(self, u, f, omega=1.0):
        return self.sweep_cells(u, f, omega, range(self.P.n_cells)).reshape(-1)
