"""GPU parity of the hybrid multigrid with the P0 subspace (Alg. 1) against
the oracle (oracle/hybrid.py), through the C ABI.

Tolerances: the coarse matrix is exact arithmetic on the same face coefficients (relative max
<= 1e-13); a V-cycle composes sweeps (local CG to 1e-13 vs the oracle's LU) and a coarse solve
(Jacobi-PCG to 1e-13 vs the oracle's dense LU): relative L2 <= 1e-9, as for a sweep; the solve
is checked against a dense solve of A u = f at the requested outer tolerance."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.hybrid import Hybrid                                    # noqa: E402
from oracle.tier_a import TierA                                     # noqa: E402
from synth import DIRICHLET, NEUMANN, make_config, make_vectors, random_problem, uniform_pm1  # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def dense_rows(P, Ah7):
    """The (7, N) stencil rows as a dense N x N matrix (face order x-, x+, y-, y+, z-, z+)."""
    N = P.n_cells
    A = np.zeros((N, N))
    step = [1, P.nx, P.nx * P.ny]
    dims = [P.nx, P.ny, P.nz]
    for T in range(N):
        co = [T % P.nx, (T // P.nx) % P.ny, T // (P.nx * P.ny)]
        A[T, T] = Ah7[0, T]
        for f in range(6):
            ax, hi = f >> 1, f & 1
            nc = co[ax] + (1 if hi else -1)
            if 0 <= nc < dims[ax]:
                A[T, T + (step[ax] if hi else -step[ax])] = Ah7[1 + f, T]
            else:
                assert Ah7[1 + f, T] == 0.0
    return A


COARSE_CASES = [
    random_problem(5, 4, 3, 1, seed=401, bc=MIXED, spread=1.5),
    random_problem(4, 3, 3, 2, seed=402, c=True, bc=MIXED, L=(1.0, 0.6, 1.4), spread=1.0),
    random_problem(3, 3, 2, 3, seed=403, alpha=1.25),
    random_problem(3, 2, 2, 4, seed=404, bc=(NEUMANN,) * 6),
    random_problem(3, 2, 2, 6, seed=405, bc=MIXED),
]


@pytest.mark.parametrize("P", COARSE_CASES, ids=[f"p{P.p}" for P in COARSE_CASES])
def test_coarse_matrix_matches_galerkin_product(P):
    ref = Hybrid(P).coarse_galerkin()
    with dg.DGContext(P) as ctx:
        got = dense_rows(P, ctx.coarse_matrix())
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


VC_CASES = [
    (random_problem(5, 4, 3, 1, seed=411, bc=MIXED, spread=1.0), 1, 1, 1.0),
    (random_problem(4, 3, 3, 2, seed=412, c=True, bc=MIXED, L=(1.0, 0.6, 1.4)), 1, 1, 0.8),
    (random_problem(3, 3, 3, 3, seed=413), 2, 1, 1.0),
    (random_problem(3, 2, 2, 4, seed=414, bc=MIXED), 0, 0, 1.0),
]


@pytest.mark.parametrize("P,npre,npost,omega", VC_CASES, ids=[f"p{c[0].p}-{c[1]}{c[2]}" for c in VC_CASES])
def test_vcycle_matches_oracle(P, npre, npost, omega):
    r = uniform_pm1(421 + P.p, 0, P.n_dof)
    ref = Hybrid(P).vcycle(r, npre, npost, omega)
    prm = dg.hybrid_params(n_pre=npre, n_post=npost, omega=omega, local_tol=1e-13, coarse_tol=1e-13)
    with dg.DGContext(P) as ctx:
        z = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.hybrid_vcycle(cuda(r), z, prm)
        got = host(z)
    assert rel(got, ref) <= 1e-9


def test_vcycle_is_linear():
    P = random_problem(4, 3, 3, 2, seed=431, bc=MIXED)
    r1, r2 = uniform_pm1(432, 0, P.n_dof), uniform_pm1(433, 0, P.n_dof)
    prm = dg.hybrid_params(local_tol=1e-13, coarse_tol=1e-13)
    with dg.DGContext(P) as ctx:
        out = []
        for r in (r1, r2, 2.0 * r1 - 3.0 * r2):
            z = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
            ctx.hybrid_vcycle(cuda(r), z, prm)
            out.append(host(z))
    assert rel(out[2], 2.0 * out[0] - 3.0 * out[1]) <= 1e-9


@pytest.mark.parametrize("P", [random_problem(4, 3, 3, 2, seed=441, bc=MIXED, spread=1.0),
                               random_problem(3, 3, 2, 3, seed=442, c=True)], ids=["p2", "p3"])
def test_solve_matches_dense_solve(P):
    f = uniform_pm1(443, 0, P.n_dof)
    ref = np.linalg.solve(TierA(P).assemble(), f)
    _, its_oracle, _ = Hybrid(P).fcg(f, tol=1e-10)
    with dg.DGContext(P) as ctx:
        u = torch.zeros(P.n_dof, dtype=torch.float64, device="cuda")
        st = ctx.hybrid_solve(u, cuda(f), dg.hybrid_params(rel_tol=1e-10))
        got = host(u)
    assert st["converged"] == 1 and st["rel_residual"] <= 1e-10
    assert abs(st["iterations"] - its_oracle) <= 2
    assert rel(got, ref) <= 1e-8


def test_solve_c2_full_size():
    """BASELINE configs[1] (32^3, Q3, 2.1M DoF): the true residual of the returned u, computed
    with dg_apply, meets the requested tolerance."""
    P = make_config("C2")
    _, f = make_vectors(P)
    with dg.DGContext(P) as ctx:
        ft = cuda(f)
        u = torch.zeros(P.n_dof, dtype=torch.float64, device="cuda")
        st = ctx.hybrid_solve(u, ft, dg.hybrid_params(rel_tol=1e-8, local_tol=1e-8, coarse_tol=1e-10))
        Au = torch.empty_like(u)
        ctx.apply(u, Au)
        res = float(torch.linalg.norm(ft - Au) / torch.linalg.norm(ft))
    assert st["converged"] == 1 and st["coarse_nonconverged"] == 0
    assert res <= 2e-8


def test_unsupported_cases_fail_loudly():
    P = random_problem(3, 2, 2, 2, seed=451, b=(1.0, 0.0, 0.0))
    with dg.DGContext(P) as ctx:
        z = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        with pytest.raises(dg.DGError):
            ctx.hybrid_vcycle(cuda(np.ones(P.n_dof)), z)
