"""Pins for the oracle's hybrid multigrid with the P0 subspace (Alg. 1; App. A.1).

The coarse matrix is pinned two ways: the closed-form finite-volume construction of App. A.1
(oracle.hybrid.Hybrid.coarse_fv) against the brute-force Galerkin product P^T A P through the
tier-B operator, and both against invariants (symmetry and SPD at b = 0, annihilated constants
under pure Neumann). The V-cycle is pinned by Galerkin orthogonality of the coarse correction,
linearity, and symmetry of the symmetric cycle; the outer flexible CG against a dense solve.
"""
import numpy as np
import pytest

from oracle.hybrid import Hybrid
from oracle.tier_a import TierA
from synth import random_problem
from synth.problem import DIRICHLET, NEUMANN

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


@pytest.mark.parametrize("p,alpha,b,c", [(1, 2.0, (0.0, 0.0, 0.0), False),
                                         (2, 1.25, (0.7, -0.4, 0.3), True),
                                         (3, 2.0, (0.0, 0.0, 0.0), True)])
def test_coarse_fv_equals_galerkin_product(p, alpha, b, c):
    """App. A.1: the rescaled FV matrix is the Galerkin product P^T A P."""
    P = random_problem(3, 2, 2, p, seed=300 + p, b=b, c=c, bc=MIXED, alpha=alpha,
                       L=(1.0, 0.7, 1.3), spread=1.2)
    H = Hybrid(P)
    G = H.coarse_galerkin()
    F = H.coarse_fv()
    assert np.abs(G - F).max() <= 1e-12 * np.abs(G).max()


def test_coarse_matrix_from_the_global_dense_matrix():
    """P^T A P with A assembled independently (tier A, 3D brute-force quadrature)."""
    P = random_problem(2, 2, 2, 2, seed=310, bc=MIXED)
    H = Hybrid(P)
    A = TierA(P).assemble()
    Pm = np.kron(np.eye(P.n_cells), np.ones((P.nd, 1)))
    assert np.abs(Pm.T @ A @ Pm - H.coarse_fv()).max() <= 1e-12 * np.abs(A).max()


def test_coarse_matrix_symmetric_spd_and_stencil():
    P = random_problem(3, 3, 2, 2, seed=311, bc=MIXED, spread=1.5)
    Ah = Hybrid(P).coarse_fv()
    assert np.abs(Ah - Ah.T).max() <= 1e-14 * np.abs(Ah).max()
    np.linalg.cholesky(Ah)
    # 7-point stencil: non-zeros only between face neighbours
    H = Hybrid(P)
    for T in range(P.n_cells):
        nbs = {T} | {H.tb.neighbour(T, a, hi) for a in range(3) for hi in (False, True)}
        for S in range(P.n_cells):
            if S not in nbs:
                assert Ah[T, S] == 0.0


def test_coarse_matrix_annihilates_constants_under_neumann():
    P = random_problem(2, 2, 3, 1, seed=312, bc=(NEUMANN,) * 6)
    Ah = Hybrid(P).coarse_fv()
    assert np.abs(Ah @ np.ones(P.n_cells)).max() <= 1e-13 * np.abs(Ah).max()


def test_coarse_correction_galerkin_orthogonal():
    """n_pre = n_post = 0: u = P A^-1 P^T r, so P^T (r - A u) = 0."""
    P = random_problem(2, 3, 2, 2, seed=313, bc=MIXED)
    H = Hybrid(P)
    r = np.random.default_rng(5).uniform(-1, 1, P.n_dof)
    u = H.vcycle(r, n_pre=0, n_post=0)
    res = H.restrict(r - H.tb.apply(u))
    assert np.abs(res).max() <= 1e-11 * np.abs(H.restrict(r)).max()


def test_vcycle_linear_and_symmetric():
    """Exact local and coarse solves: the cycle is a fixed linear map, symmetric for b = 0 with
    the same number of pre- and post-sweeps (block Jacobi is self-adjoint)."""
    P = random_problem(2, 2, 2, 2, seed=314, bc=MIXED)
    H = Hybrid(P)
    Ah = H.coarse_galerkin()
    rng = np.random.default_rng(6)
    r1, r2 = rng.uniform(-1, 1, (2, P.n_dof))
    V = lambda r: H.vcycle(r, 1, 1, 0.8, Ah)   # noqa: E731
    v1, v2 = V(r1), V(r2)
    assert np.linalg.norm(V(2.0 * r1 - 3.0 * r2) - (2.0 * v1 - 3.0 * v2)) <= 1e-11 * np.linalg.norm(v1)
    assert abs(v1 @ r2 - r1 @ v2) <= 1e-11 * abs(v1 @ r2)


def test_fcg_solves_the_system():
    P = random_problem(3, 2, 2, 2, seed=315, bc=MIXED, spread=1.0)
    H = Hybrid(P)
    f = np.random.default_rng(7).uniform(-1, 1, P.n_dof)
    u, its, hist = H.fcg(f, tol=1e-10)
    A = TierA(P).assemble()
    ref = np.linalg.solve(A, f)
    assert hist[-1] <= 1e-10 and its < 40
    assert np.linalg.norm(u - ref) <= 1e-8 * np.linalg.norm(ref)
