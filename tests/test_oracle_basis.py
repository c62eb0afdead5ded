"""Pins for the oracle's 1D tables and face parameters (closed forms and worked values)."""
import json
import os

import numpy as np
import pytest

from oracle.basis import (face_weights, gauss_rule, harmonic_average, lagrange_derivs,
                          lagrange_values, lobatto_nodes, upwind)
from oracle.tier_b import TierB
from synth import make_config, splitmix64, uniform_pm1, normal, random_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_values():
    # SplitMix64 (Steele, Lea, Flood 2014) from state 0: published first outputs
    assert [int(x) for x in splitmix64(0, 0, 3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                     0x06C45D188009454F]


def test_streams_are_counter_based_and_in_range():
    a = uniform_pm1(5, 0, 1000)
    b = uniform_pm1(5, 300, 200)
    assert np.array_equal(a[300:500], b)
    assert a.min() >= -1.0 and a.max() < 1.0
    z = normal(9, 0, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01


def test_lobatto_closed_forms():
    # S:115 (p=3) and symmetry (p=2 midpoint); nodes are the roots of (1-x^2) P_p'
    assert np.allclose(lobatto_nodes(1), [0, 1], atol=0, rtol=0)
    assert np.allclose(lobatto_nodes(2), [0, 0.5, 1], atol=1e-16)
    s = 1 / np.sqrt(5)
    assert np.allclose(lobatto_nodes(3), [0, (1 - s) / 2, (1 + s) / 2, 1], atol=1e-15)
    # p=4: interior roots 0.5 +- sqrt(21)/14 on [0,1]
    r = np.sqrt(21) / 14
    assert np.allclose(lobatto_nodes(4), [0, 0.5 - r, 0.5, 0.5 + r, 1], atol=1e-15)
    for p in range(1, 8):
        z = lobatto_nodes(p)
        assert np.all(np.diff(z) > 0) and np.allclose(z + z[::-1], 1.0, atol=1e-15)


def test_gauss_rule_closed_forms_and_exactness():
    x, w = gauss_rule(2)
    assert np.allclose(x, [0.5 - 1 / (2 * np.sqrt(3)), 0.5 + 1 / (2 * np.sqrt(3))], atol=1e-16)
    assert np.allclose(w, [0.5, 0.5], atol=1e-16)
    x, w = gauss_rule(1)
    assert np.allclose(x, [0.5]) and np.allclose(w, [1.0])
    for m in range(1, 10):
        x, w = gauss_rule(m)
        for d in range(2 * m):
            assert abs(w @ x ** d - 1.0 / (d + 1)) < 1e-14
        # degree 2m is NOT exact (the rule is exactly of order 2m-1)
        assert abs(w @ x ** (2 * m) - 1.0 / (2 * m + 1)) > 1e-12


def test_lagrange_nodal_partition_of_unity():
    for p in range(1, 8):
        z = lobatto_nodes(p)
        assert np.allclose(lagrange_values(z, z), np.eye(p + 1), atol=1e-13)
        x = np.linspace(0, 1, 17)
        assert np.allclose(lagrange_values(z, x).sum(1), 1.0, atol=1e-13)
        assert np.allclose(lagrange_derivs(z, x).sum(1), 0.0, atol=1e-11)
        # derivative against a central difference of the values
        hh = 1e-6
        fd = (lagrange_values(z, x[1:-1] + hh) - lagrange_values(z, x[1:-1] - hh)) / (2 * hh)
        assert np.allclose(fd, lagrange_derivs(z, x[1:-1]), atol=1e-6 * (p + 1) ** 3)


def test_endpoint_derivative_closed_form():
    # theta_p'(1) = -theta_0'(0) = p(p+1)/2 on [0,1] (GL nodal basis)
    for p in range(1, 8):
        z = lobatto_nodes(p)
        d1 = lagrange_derivs(z, [1.0])[0]
        d0 = lagrange_derivs(z, [0.0])[0]
        assert abs(d1[-1] - p * (p + 1) / 2) < 1e-10 * p * p
        assert abs(d0[0] + p * (p + 1) / 2) < 1e-10 * p * p


def test_mass_row_sums_are_lobatto_weights():
    # the exact mass matrix's row sums are int theta_i = GLL weights; p=2: 1/6, 2/3, 1/6
    P = random_problem(1, 1, 1, 2, seed=1)
    assert np.allclose(TierB(P).Mh.sum(1), [1 / 6, 2 / 3, 1 / 6], atol=1e-15)
    P = random_problem(1, 1, 1, 3, seed=1)
    assert np.allclose(TierB(P).Mh.sum(1), [1 / 12, 5 / 12, 5 / 12, 1 / 12], atol=1e-15)


def test_face_parameter_worked_values():
    # S:187-198 worked values
    assert harmonic_average(1.0, 3.0) == 1.5
    assert harmonic_average(2.0, 2.0) == 2.0
    assert harmonic_average(0.0, 5.0) == 0.0
    assert harmonic_average(0.0, 0.0) == 0.0
    assert face_weights(1.0, 3.0) == (0.75, 0.25)
    assert face_weights(0.0, 0.0) == (0.5, 0.5)
    assert upwind(2, 5, 1) == 2 and upwind(2, 5, -1) == -5 and upwind(2, 5, 0) == 0


def test_penalty_worked_values():
    # K=I, h=0.25, p=1, alpha=1.25 -> gamma = 15;  C1: alpha=2, p=2, h=1/8 -> 128
    P = random_problem(4, 4, 4, 1, seed=1, aniso=False, spread=0.0, alpha=1.25)
    assert abs(TierB(P).face_params(21, 0, True)[3] - 15.0) < 1e-12
    C1 = make_config("C1")
    assert abs(TierB(C1).face_params(100, 2, True)[3] - 128.0) < 1e-12
    assert abs(TierB(C1).face_params(0, 0, False)[3] - 128.0) < 1e-12   # Dirichlet, K=1


def test_config_shapes():
    with open(os.path.join(GOLDEN, "configs.json")) as fh:
        gold = json.load(fh)
    for name, g in [(k, v) for k, v in gold.items() if not k.startswith("_")]:
        P = make_config(name)
        assert [P.nx, P.ny, P.nz, P.p] == g["mesh_p"], name
        assert P.n_dof == g["dofs"], name
        # face counts: interior and boundary
        nx, ny, nz = P.nx, P.ny, P.nz
        assert (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1) == g["interior_faces"]
        assert 2 * (ny * nz + nx * nz + nx * ny) == g["boundary_faces"]
    C5 = make_config("C5")
    lk = np.log10(C5.K[:, 0])
    assert lk.min() >= -3.0 - 1e-12 and lk.max() <= 4.3 + 1e-12
    assert np.allclose(C5.K[:, 2], 0.1 * C5.K[:, 0])
