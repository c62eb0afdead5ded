"""GPU parity of the Thomas-preconditioned local BiCGStab: the
sweep with the tridiagonal part of D_T (DoF order) as preconditioner against the oracle's exact
LU sweep (relative L2 <= 1e-9, local tolerance 1e-12), and its effect in the strongly convection-
dominated regime where the diagonal preconditioner stalls."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.tier_b import TierB                                     # noqa: E402
from synth import DIRICHLET, NEUMANN, random_problem, uniform_pm1   # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def sweep(P, method, u, f, max_it=1000):
    with dg.DGContext(P) as ctx:
        ctx.set_local_solver(method, max_it)
        ut = cuda(u)
        ctx.sweep(ut, cuda(f), 1.0, 1e-12)
        st = ctx.stats()
        torch.cuda.synchronize()
        return ut.cpu().numpy(), st


CASES = [random_problem(5, 4, 3, p, seed=800 + p, b=(1.0, -0.5, 0.25), c=True, bc=MIXED, L=(1.0, 0.6, 1.4))
         for p in (1, 2, 3, 4)] + [random_problem(3, 3, 2, 3, seed=810, spread=1.0)]


@pytest.mark.parametrize("P", CASES, ids=[f"p{P.p}{'-conv' if any(P.b) else ''}" for P in CASES])
def test_thomas_sweep_matches_oracle(P):
    u, f = uniform_pm1(820 + P.p, 0, P.n_dof), uniform_pm1(830 + P.p, 0, P.n_dof)
    ref = TierB(P).sweep(u, f, 1.0)
    got, st = sweep(P, dg.DG_LOCAL_BICGSTAB_THOMAS, u, f)
    assert st["n_nonconverged"] == 0
    assert rel(got, ref) <= 1e-9


@pytest.mark.parametrize("b", [(1.0, 0.0, 0.0), (1.0, 0.5, 0.3)])
def test_convection_dominated_blocks(b):
    """eps = 1e-6, |b| ~ 1, h = 1/4: cell Peclet ~ 2.5e5 (the paper's test uses 2000). The
    tridiagonal preconditioner converges every block to 1e-12 and matches the LU sweep."""
    P = random_problem(4, 4, 4, 3, seed=840, b=b, spread=0.0)
    P.K = np.asarray(P.K) * 1e-6
    u, f = uniform_pm1(841, 0, P.n_dof), uniform_pm1(842, 0, P.n_dof)
    ref = TierB(P).sweep(u, f, 1.0)
    got_t, st_t = sweep(P, dg.DG_LOCAL_BICGSTAB_THOMAS, u, f)
    _, st_j = sweep(P, dg.DG_LOCAL_BICGSTAB, u, f, max_it=200)
    assert st_t["n_nonconverged"] == 0
    assert rel(got_t, ref) <= 1e-9
    assert st_t["it_max"] < st_j["it_max"] or st_j["n_nonconverged"] > 0
