"""Hybrid multigrid with the P0 subspace (Alg. 1): the CPU oracle of SURVEY 8(f) NEXT-1.

ORACLE (test infrastructure only; never imported by the product path).

  prolongation  P|_T = (1, ..., 1)^T                       (partition of unity)
  restriction   R = P^T  (cell sums of the DoF values)
  coarse matrix A^ = P^T A P (the Galerkin product, eq. galerkin_product),
                computed here by brute force from the tier-B operator, and in closed form
                (`coarse_fv`) as the rescaled finite-volume matrix of App. A.1,
                the two pinned equal in tests/test_oracle_hybrid.py
  V-cycle       Alg. 1: n_pre block-Jacobi sweeps from u0 = 0, residual, restriction, coarse
                solve (exact, dense LU here: the paper's AMG V-cycle is out of scope and the
                GPU path solves A^ by Jacobi-PCG to a tight tolerance), prolongation,
                n_post sweeps
  outer solver  flexible preconditioned CG (the V-cycle as preconditioner), relative
                residual stopping rule ||r|| <= tol ||r_0||

Reading (DESIGN.md §2 #24): App. A.1 states the boundary rescaling factor as 2 alpha p(p+d-1)
together with 1/||x^-(F) - x(F)|| = |F|/(2|T|); on the uniform box ||x^- - x(F)|| = h/2, i.e.
1/||.|| = 2|F|/|T|, and the factor that reproduces P^T A P is alpha p(p+d-1)/2. The definition
A^ = P^T A P decides; `coarse_fv` uses the cell-centre distances as written and the factor that
makes it equal to the Galerkin product.
"""
from __future__ import annotations

import numpy as np

from synth.problem import DIRICHLET, Problem
from .basis import harmonic_average
from .tier_b import TierB


class Hybrid:
    def __init__(self, P: Problem, tb: TierB | None = None):
        self.P = P
        self.tb = tb if tb is not None else TierB(P)
        self.nd = self.tb.nd
        self.N = P.n_cells

    # ---- transfer -------------------------------------------------
    def prolongate(self, uh):
        return np.repeat(np.asarray(uh, dtype=np.float64), self.nd)

    def restrict(self, r):
        return np.asarray(r, dtype=np.float64).reshape(self.N, self.nd).sum(axis=1)

    # ---- coarse matrix ----------------------------------------------------------
    def coarse_galerkin(self):
        """A^ = P^T A P by applying the tier-B operator to every prolongated unit vector."""
        N = self.N
        Ah = np.zeros((N, N))
        for j in range(N):
            e = np.zeros(N)
            e[j] = 1.0
            Ah[:, j] = self.restrict(self.tb.apply(self.prolongate(e)))
        return Ah

    def coarse_fv(self):
        """App. A.1 (eq. p0_matrix): cell-centred finite volumes with the upwind
        convective flux, the reaction c|T|, the harmonic-mean diffusive flux over the
        centre distance (interior) and the one-sided flux over the centre-face distance
        (Dirichlet), rescaled by alpha p(p+d-1) (interior) and alpha p(p+d-1)/2 (boundary,
        reading #24) to equal the Galerkin product on the uniform box."""
        P, tb = self.P, self.tb
        N = self.N
        h = np.asarray(P.h, dtype=np.float64)
        vol = h[0] * h[1] * h[2]
        area = [h[1] * h[2], h[0] * h[2], h[0] * h[1]]
        scale = P.alpha * P.p * (P.p + 2)
        Ah = np.zeros((N, N))
        for T in range(N):
            Ah[T, T] += tb.c[T] * vol
            for axis in range(3):
                for hi in (False, True):
                    nb = tb.neighbour(T, axis, hi)
                    F = area[axis]
                    if nb is None:
                        if P.bc[2 * axis + (1 if hi else 0)] != DIRICHLET:
                            continue
                        bnu = tb.b[T, axis] * (1.0 if hi else -1.0)
                        dist = 0.5 * h[axis]                     # ||x^-(F) - x(F)||
                        Ah[T, T] += max(bnu, 0.0) * F           # Phi(psi, 0, nu.b) [psi]
                        Ah[T, T] += 0.5 * scale * tb.K[T, axis] / dist * F
                        continue
                    # interior face, seen from T (nu = outward normal of T): row T only
                    bnu = 0.5 * (tb.b[T, axis] + tb.b[nb, axis]) * (1.0 if hi else -1.0)
                    Ah[T, T] += max(bnu, 0.0) * F                # outflow: T's own value
                    Ah[T, nb] += min(bnu, 0.0) * F               # inflow: the neighbour's value
                    dist = h[axis]                               # ||x^-(F) - x^+(F)||
                    s = scale * harmonic_average(tb.K[T, axis], tb.K[nb, axis]) / dist * F
                    Ah[T, T] += s
                    Ah[T, nb] -= s
        return Ah

    # ---- Alg. 1 -----------------------------------------------------------------
    def vcycle(self, f, n_pre=1, n_post=1, omega=1.0, Ah=None):
        """One hybrid V-cycle with u0 = 0 (Alg. 1 lines 1-6), exact coarse solve."""
        tb = self.tb
        Ah = self.coarse_galerkin() if Ah is None else Ah
        u = np.zeros(self.N * self.nd)
        for _ in range(n_pre):
            u = tb.sweep(u, f, omega)
        r = f - tb.apply(u)
        uh = np.linalg.solve(Ah, self.restrict(r))
        u = u + self.prolongate(uh)
        for _ in range(n_post):
            u = tb.sweep(u, f, omega)
        return u

    def fcg(self, f, u0=None, tol=1e-10, max_it=200, n_pre=1, n_post=1, omega=1.0):
        """Flexible PCG (beta = z_new.(r_new - r_old) / z_old.r_old) preconditioned by the
        V-cycle; returns (u, iterations, relative residual history)."""
        tb = self.tb
        Ah = self.coarse_galerkin()
        u = np.zeros(self.N * self.nd) if u0 is None else np.array(u0, dtype=np.float64)
        r = f - tb.apply(u)
        r0 = np.linalg.norm(r)
        hist = [1.0]
        if r0 == 0.0:
            return u, 0, hist
        z = self.vcycle(r, n_pre, n_post, omega, Ah)
        p = z.copy()
        zr = z @ r
        for it in range(1, max_it + 1):
            q = tb.apply(p)
            alpha = zr / (p @ q)
            u = u + alpha * p
            r_new = r - alpha * q
            hist.append(np.linalg.norm(r_new) / r0)
            if hist[-1] <= tol:
                return u, it, hist
            z = self.vcycle(r_new, n_pre, n_post, omega, Ah)
            beta = (z @ (r_new - r)) / zr
            zr = z @ r_new
            p = z + beta * p
            r = r_new
        return u, max_it, hist
