"""GPU edge cases against the oracle: degenerate mesh shapes (one cell thick in one or two
directions, a single row of groups), zero diffusion in some cells (the degenerate-weight
convention, DESIGN reading #7), pure Neumann constants, extreme coefficient contrast, and the
convection sign cases — apply (<= 1e-12), sweeps (<= 1e-9), through the C ABI."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.tier_b import TierB                                     # noqa: E402
from synth import DIRICHLET, NEUMANN, random_problem, uniform_pm1  # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def run(P, u, f, omega=1.0):
    with dg.DGContext(P) as ctx:
        Au = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.apply(cuda(u), Au)
        ut = cuda(u)
        ctx.sweep(ut, cuda(f), omega, 1e-12)
        st = ctx.stats()
        torch.cuda.synchronize()
        return Au.cpu().numpy(), ut.cpu().numpy(), st


SHAPES = [(40, 1, 1), (1, 37, 1), (1, 1, 33), (9, 7, 1), (1, 6, 5), (33, 2, 1)]
CASES = [(s, p) for s in SHAPES for p in (1, 3)] + [((5, 1, 4), 2), ((1, 3, 2), 4), ((7, 1, 1), 6)]


@pytest.mark.parametrize("shape,p", CASES, ids=[f"{s[0]}x{s[1]}x{s[2]}-p{p}" for s, p in CASES])
def test_degenerate_shapes(shape, p):
    P = random_problem(*shape, p, seed=950 + p, bc=MIXED, L=(1.0, 0.7, 1.3))
    u, f = uniform_pm1(951, 0, P.n_dof), uniform_pm1(952, 0, P.n_dof)
    tb = TierB(P)
    Au, us, st = run(P, u, f)
    assert rel(Au, tb.apply(u)) <= 1e-12
    assert st["n_nonconverged"] == 0
    assert rel(us, tb.sweep(u, f, 1.0)) <= 1e-9


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_zero_diffusion_cells(p):
    """K = 0 in a third of the cells (harmonic mean 0, weights 1/2, gamma = 0 on their faces)
    with a reaction term so every block stays SPD."""
    P = random_problem(4, 3, 3, p, seed=960 + p, c=True, bc=MIXED)
    K = np.array(P.K)
    K[::3] = 0.0
    P.K = K
    u, f = uniform_pm1(961, 0, P.n_dof), uniform_pm1(962, 0, P.n_dof)
    tb = TierB(P)
    Au, us, st = run(P, u, f)
    assert rel(Au, tb.apply(u)) <= 1e-12
    assert st["n_nonconverged"] == 0
    assert rel(us, tb.sweep(u, f, 1.0)) <= 1e-9


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_pure_neumann_annihilates_constants(p):
    P = random_problem(4, 3, 2, p, seed=970 + p, bc=(NEUMANN,) * 6)
    with dg.DGContext(P) as ctx:
        one = torch.ones(P.n_dof, dtype=torch.float64, device="cuda")
        out = torch.empty_like(one)
        ctx.apply(one, out)
        # relative to the operator's scale (the apply of a random vector)
        v = cuda(uniform_pm1(971, 0, P.n_dof))
        ref = torch.empty_like(one)
        ctx.apply(v, ref)
        assert float(out.abs().max()) <= 1e-12 * float(ref.abs().max())


@pytest.mark.parametrize("p", [2, 3])
def test_extreme_contrast(p):
    """K spanning ~1e-5 .. 1e5 between neighbours (beyond C3's 6.6e-5 .. 1.2e4)."""
    P = random_problem(5, 4, 3, p, seed=980 + p, spread=4.0)
    u, f = uniform_pm1(981, 0, P.n_dof), uniform_pm1(982, 0, P.n_dof)
    tb = TierB(P)
    Au, us, st = run(P, u, f)
    assert rel(Au, tb.apply(u)) <= 1e-12
    assert st["n_nonconverged"] == 0
    assert rel(us, tb.sweep(u, f, 1.0)) <= 1e-9


@pytest.mark.parametrize("b", [(-1.0, 0.0, 0.0), (0.0, -2.0, 0.5), (0.3, 0.3, -0.7)])
def test_convection_directions(b):
    """Negative and mixed-sign b: the upwind side flips per face."""
    P = random_problem(4, 3, 3, 2, seed=990, b=b, c=True, bc=MIXED)
    u, f = uniform_pm1(991, 0, P.n_dof), uniform_pm1(992, 0, P.n_dof)
    tb = TierB(P)
    Au, us, st = run(P, u, f, 0.8)
    assert rel(Au, tb.apply(u)) <= 1e-12
    assert st["n_nonconverged"] == 0
    assert rel(us, tb.sweep(u, f, 0.8)) <= 1e-9


def test_isotropic_scalar_k_input():
    """k_components = 1 (scalar K per cell) goes through the same kernels as the diagonal case."""
    P = random_problem(3, 3, 3, 3, seed=995, aniso=False)
    assert np.asarray(P.K).ndim == 1
    u, f = uniform_pm1(996, 0, P.n_dof), uniform_pm1(997, 0, P.n_dof)
    tb = TierB(P)
    Au, us, _ = run(P, u, f)
    assert rel(Au, tb.apply(u)) <= 1e-12
    assert rel(us, tb.sweep(u, f, 1.0)) <= 1e-9


def test_one_call_stats_forms_equal_the_two_call_forms():
    """dg_block_jacobi_sweep_stats / dg_local_block_solve_stats (SURVEY 8(b)'s signatures) give
    the bits of the plain calls and the statistics dg_get_stats reports after them."""
    P = random_problem(4, 3, 3, 3, seed=61, spread=1.0)
    u, f = uniform_pm1(62, 0, P.n_dof), uniform_pm1(63, 0, P.n_dof)
    with dg.DGContext(P) as ctx:
        a, b = cuda(u), cuda(u)
        ft = cuda(f)
        ctx.sweep(a, ft, 0.9, 1e-12)
        st_two = ctx.stats()
        st_one = ctx.sweep_stats(b, ft, 0.9, 1e-12)
        assert torch.equal(a, b) and st_one == st_two and st_one["n_cells"] == P.n_cells
        assert st_one["it_min"] >= 1 and st_one["n_nonconverged"] == 0
        da, db = torch.empty_like(a), torch.empty_like(a)
        ctx.local_block_solve(ft, da, 1e-12)
        st_two = ctx.stats()
        st_one = ctx.local_block_solve_stats(ft, db, 1e-12)
        assert torch.equal(da, db) and st_one == st_two
