"""Pins for the oracle's block-Jacobi sweep (Alg. 2) and exact local solves."""
import numpy as np
import pytest

from oracle.tier_a import TierA
from oracle.tier_b import TierB
from synth import random_problem

CASES = [((0.0, 0.0, 0.0), False), ((1.0, 0.5, 0.25), True)]


@pytest.mark.parametrize("b,c", CASES)
def test_local_solve_matches_dense_block_of_tier_a(b, c):
    """D_T = A_{T,T} taken from the tier-A global matrix; LU solve residual."""
    P = random_problem(2, 2, 2, 2, seed=61, b=b, c=c)
    A = TierA(P).assemble()
    tb = TierB(P)
    nd = P.nd
    d = np.random.default_rng(0).uniform(-1, 1, P.n_dof)
    du = tb.local_solve(d)
    for t in range(P.n_cells):
        s = slice(t * nd, (t + 1) * nd)
        assert np.linalg.norm(A[s, s] @ du[t] - d[s]) <= 1e-12 * np.linalg.norm(d[s])
    assert np.abs(tb.local_solve(np.zeros(P.n_dof))).max() == 0.0


@pytest.mark.parametrize("b,c", CASES)
def test_sweep_fixed_point(b, c):
    """u = A^{-1} f is a fixed point of every block-Jacobi sweep."""
    P = random_problem(2, 3, 2, 2, seed=62, b=b, c=c)
    A = TierA(P).assemble()
    f = np.random.default_rng(1).uniform(-1, 1, P.n_dof)
    u = np.linalg.solve(A, f)
    assert np.linalg.norm(TierB(P).sweep(u, f, 0.7) - u) <= 1e-10 * np.linalg.norm(u)


@pytest.mark.parametrize("b,c", CASES)
def test_sweep_from_zero_is_block_inverse(b, c):
    """u = 0, omega = 1: one sweep returns D^{-1} f, D from the tier-A matrix."""
    P = random_problem(2, 2, 2, 1, seed=63, b=b, c=c)
    A = TierA(P).assemble()
    nd = P.nd
    f = np.random.default_rng(2).uniform(-1, 1, P.n_dof)
    out = TierB(P).sweep(np.zeros(P.n_dof), f, 1.0)
    for t in range(P.n_cells):
        s = slice(t * nd, (t + 1) * nd)
        assert np.allclose(out[s], np.linalg.solve(A[s, s], f[s]), rtol=1e-11, atol=1e-13)


def test_single_cell_sweep_solves_system():
    """On a 1-cell mesh D_T = A, so one exact sweep with omega=1 gives A u = f."""
    P = random_problem(1, 1, 1, 3, seed=64, b=(0.4, -0.2, 0.1), c=True)
    A = TierA(P).assemble()
    rng = np.random.default_rng(3)
    u0, f = rng.uniform(-1, 1, P.n_dof), rng.uniform(-1, 1, P.n_dof)
    u1 = TierB(P).sweep(u0, f, 1.0)
    assert np.linalg.norm(A @ u1 - f) <= 1e-11 * np.linalg.norm(f)


def test_sweep_linearity():
    """sweep(a u, a f) = a sweep(u, f) and additivity in (u, f)."""
    P = random_problem(2, 2, 2, 2, seed=65, b=(0.3, 0.0, 0.0))
    tb = TierB(P)
    rng = np.random.default_rng(4)
    u1, f1, u2, f2 = (rng.uniform(-1, 1, P.n_dof) for _ in range(4))
    s = tb.sweep(u1 + 2 * u2, f1 + 2 * f2, 0.8)
    assert np.allclose(s, tb.sweep(u1, f1, 0.8) + 2 * tb.sweep(u2, f2, 0.8), rtol=1e-11, atol=1e-12)


def test_sweep_contracts_on_poisson():
    """Block-Jacobi is a convergent smoother on SPD Poisson with omega < 1: the error in the
    energy norm decreases monotonically (sanity of the Alg. 2 update direction)."""
    P = random_problem(3, 3, 3, 1, seed=66, aniso=False, spread=0.0)
    A = TierB(P).assemble()
    f = np.random.default_rng(5).uniform(-1, 1, P.n_dof)
    x = np.linalg.solve(A, f)
    u = np.zeros(P.n_dof)
    tb = TierB(P)
    prev = np.inf
    for _ in range(4):
        u = tb.sweep(u, f, 0.7)
        e = u - x
        en = e @ A @ e
        assert en < prev
        prev = en
