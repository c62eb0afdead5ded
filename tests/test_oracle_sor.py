"""Pins for the oracle's red-black block SOR / SSOR (Alg. 3)."""
import numpy as np
import pytest

from oracle import sor
from oracle.tier_a import TierA
from oracle.tier_b import TierB
from synth import random_problem
from synth.problem import DIRICHLET, NEUMANN

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


@pytest.mark.parametrize("b,omega", [((0.0, 0.0, 0.0), 1.0), ((0.8, -0.3, 0.2), 1.3)])
def test_coloured_sweep_is_alg3_in_red_black_order(b, omega):
    """Alg. 3 literally (off-diagonal defect, (1 - omega) u + omega du) in the red-black order
    equals the coloured form u + omega D^-1 (f - A u) per colour (reading #17)."""
    P = random_problem(3, 3, 2, 2, seed=501, b=b, c=True, bc=MIXED)
    tb = TierB(P)
    rng = np.random.default_rng(8)
    u, f = rng.uniform(-1, 1, (2, P.n_dof))
    ref = sor.alg3(tb, u, f, omega, sor.red_black_order(tb))
    got = sor.sor_sweep(tb, u, f, omega)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    # the order inside a colour is immaterial (same-colour cells do not touch)
    order = sor.red_black_order(tb)
    nred = sum(1 for c in order if sor.colour(tb, c) == 0)
    shuffled = list(rng.permutation(order[:nred])) + list(rng.permutation(order[nred:]))
    assert np.linalg.norm(sor.alg3(tb, u, f, omega, shuffled) - ref) <= 1e-12 * np.linalg.norm(ref)


def test_ssor_is_forward_then_backward():
    P = random_problem(3, 2, 3, 1, seed=502, bc=MIXED)
    tb = TierB(P)
    rng = np.random.default_rng(9)
    u, f = rng.uniform(-1, 1, (2, P.n_dof))
    fwd = sor.alg3(tb, u, f, 1.1, sor.red_black_order(tb))
    ref = sor.alg3(tb, fwd, f, 1.1, sor.red_black_order(tb, reverse=True))
    got = sor.sor_sweep(tb, u, f, 1.1, symmetric=True)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_fixed_point_and_symmetric_ssor_map():
    P = random_problem(2, 3, 2, 2, seed=503, bc=MIXED)
    tb = TierB(P)
    A = TierA(P).assemble()
    rng = np.random.default_rng(10)
    f = rng.uniform(-1, 1, P.n_dof)
    x = np.linalg.solve(A, f)
    assert np.linalg.norm(sor.sor_sweep(tb, x, f, 1.2) - x) <= 1e-10 * np.linalg.norm(x)
    # b = 0: f -> SSOR(0, f) is a symmetric linear map (W^-1 of P:612-614 is symmetric)
    f1, f2 = rng.uniform(-1, 1, (2, P.n_dof))
    z = np.zeros(P.n_dof)
    s1 = sor.sor_sweep(tb, z, f1, 0.9, symmetric=True)
    s2 = sor.sor_sweep(tb, z, f2, 0.9, symmetric=True)
    assert abs(s1 @ f2 - f1 @ s2) <= 1e-12 * abs(s1 @ f2)


def test_gauss_seidel_converges_faster_than_jacobi():
    """Poisson, omega = 1: the red-black block Gauss-Seidel error contracts faster than block
    Jacobi (spectral radius rho_GS = rho_J^2 for this 2-cyclic ordering)."""
    P = random_problem(4, 3, 3, 1, seed=504, aniso=False, spread=0.0)
    tb = TierB(P)
    A = TierA(P).assemble()
    f = np.random.default_rng(11).uniform(-1, 1, P.n_dof)
    x = np.linalg.solve(A, f)
    uj = ug = np.zeros(P.n_dof)
    for _ in range(6):
        uj = tb.sweep(uj, f, 1.0)
        ug = sor.sor_sweep(tb, ug, f, 1.0)
    ej, eg = np.linalg.norm(uj - x), np.linalg.norm(ug - x)
    assert eg < 0.5 * ej
