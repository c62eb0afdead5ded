"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/dg.h declares,
its host-built 1D tables match the oracle's independent ones, and invalid descriptors are
rejected before any device work (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1805_11930_b200 as pkg
from paper_1805_11930_b200 import dg as dgb
from oracle.basis import gauss_rule, lagrange_derivs, lagrange_values, lobatto_nodes
from synth import random_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1805_11930_b200.build import build
    build()
    return pkg.load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    decl = declared_symbols()
    assert len(decl) >= 15
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(dgb.EXPORTS) == decl
    assert b"sm_100a" in lib.dg_version()


@pytest.mark.parametrize("p", range(1, 8))
def test_tables_match_oracle(lib, p):
    """GL nodes, Gauss rule, A = theta_j(xi_q), collocation derivative D (D A = G), face mass M,
    end-point derivatives — built in C++ by Newton iterations, checked against the oracle's
    numpy.polynomial-based construction."""
    t = pkg.tables(p)
    z = lobatto_nodes(p)
    xq, wq = gauss_rule(p + 1)
    assert np.allclose(t["z"], z, atol=1e-15, rtol=0)
    assert np.allclose(t["xq"], xq, atol=1e-15, rtol=0)
    assert np.allclose(t["wq"], wq, atol=1e-15, rtol=0)
    V = lagrange_values(z, xq)
    G = lagrange_derivs(z, xq)
    assert np.allclose(t["A"], V, atol=1e-13)
    assert np.allclose(t["D"] @ t["A"], G, atol=1e-11 * (p + 1) ** 2)
    assert np.allclose(t["M"], np.einsum("q,qi,qj->ij", wq, V, V), atol=1e-14)
    assert np.allclose(t["d0"], lagrange_derivs(z, [0.0])[0], atol=1e-11)
    assert np.allclose(t["d1"], lagrange_derivs(z, [1.0])[0], atol=1e-11)


def _desc(P, **kw):
    K = np.ascontiguousarray(P.K3())
    d = dgb.dg_desc()
    d.nx, d.ny, d.nz, d.Lx, d.Ly, d.Lz = P.nx, P.ny, P.nz, P.Lx, P.Ly, P.Lz
    d.bc[:] = list(P.bc)
    d.p, d.alpha, d.k_components = P.p, P.alpha, 3
    d.K = K.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    d.nranks = 1
    for k, v in kw.items():
        setattr(d, k, v)
    return d, K


@pytest.mark.parametrize("field,value", [("p", 0), ("p", 8), ("nx", 0), ("Lx", 0.0),
                                         ("Lz", -1.0), ("k_components", 2), ("nranks", 0),
                                         ("halo_mode", 7)])
def test_invalid_descriptors_rejected(lib, field, value):
    P = random_problem(2, 2, 2, 2, seed=1)
    d, keep = _desc(P, **{field: value})
    h = ctypes.c_void_p()
    assert lib.dg_create(ctypes.byref(d), ctypes.byref(h)) == dgb.DG_ERR_INVALID
    assert h.value is None
    assert len(lib.dg_last_error()) > 0


def test_negative_coefficients_and_bad_ranks_rejected(lib):
    P = random_problem(2, 2, 2, 2, seed=1)
    P.K = -np.ones(P.n_cells)
    d, keep = _desc(P)
    h = ctypes.c_void_p()
    assert lib.dg_create(ctypes.byref(d), ctypes.byref(h)) == dgb.DG_ERR_INVALID
    P = random_problem(2, 2, 2, 2, seed=1)
    d, keep = _desc(P, nranks=3)   # more ranks than z-layers
    assert lib.dg_create(ctypes.byref(d), ctypes.byref(h)) == dgb.DG_ERR_INVALID
    d, keep = _desc(P, nranks=2, rank=0, halo_mode=0)   # NCCL mode without an id
    assert lib.dg_create(ctypes.byref(d), ctypes.byref(h)) == dgb.DG_ERR_INVALID


def test_null_arguments(lib):
    h = ctypes.c_void_p()
    assert lib.dg_create(None, ctypes.byref(h)) == dgb.DG_ERR_INVALID
    assert lib.dg_apply(None, None, None, None) == dgb.DG_ERR_INVALID
    assert lib.dg_destroy(None) == dgb.DG_ERR_INVALID
    assert lib.dg_tables(9, (ctypes.c_double * 400)()) == dgb.DG_ERR_INVALID


def test_valid_descriptor_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    P = random_problem(2, 2, 2, 2, seed=1)
    d, keep = _desc(P)
    h = ctypes.c_void_p()
    code = lib.dg_create(ctypes.byref(d), ctypes.byref(h))
    assert code in (dgb.DG_ERR_CUDA, dgb.DG_ERR_UNSUPPORTED)
    assert h.value is None
