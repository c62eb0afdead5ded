"""GPU parity of the restarted local GMRES (the paper's local Krylov method
for the convection test, with the diagonal or the tridiagonal preconditioner,
P:909-918), Krylov basis in tensor memory: block-Jacobi and red-black SOR sweeps and the batched
local solve against the oracle's exact LU (relative L2 <= 1e-9 with local tolerance 1e-12),
restarts, the iteration cap, and the convection-dominated regime."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import sor                                              # noqa: E402
from oracle.tier_b import TierB                                     # noqa: E402
from synth import DIRICHLET, NEUMANN, random_problem, uniform_pm1   # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)
METHODS = [("gmres", dg.DG_LOCAL_GMRES), ("gmres-thomas", dg.DG_LOCAL_GMRES_THOMAS)]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def sweep(P, method, u, f, omega=1.0, max_it=1000):
    with dg.DGContext(P) as ctx:
        ctx.set_local_solver(method, max_it)
        ut = cuda(u)
        ctx.sweep(ut, cuda(f), omega, 1e-12)
        st = ctx.stats()
        torch.cuda.synchronize()
        return ut.cpu().numpy(), st


# several CTAs with a ragged last group (p = 1: 64 cells per CTA, p = 2: 40, p = 3: 32)
CASES = [random_problem(*{1: (9, 5, 3), 2: (7, 4, 3), 3: (5, 4, 3)}[p], p, seed=1100 + p,
                        b=(1.0, -0.5, 0.25), c=True, bc=MIXED, L=(1.0, 0.6, 1.4)) for p in (1, 2, 3)]
CASES += [random_problem(4, 3, 3, 3, seed=1110, spread=1.5),                    # SPD blocks
          random_problem(5, 3, 2, 2, seed=1111, b=(-2.0, 1.0, 0.0), bc=(NEUMANN,) * 6)]


@pytest.mark.parametrize("name,method", METHODS, ids=[m[0] for m in METHODS])
@pytest.mark.parametrize("P", CASES, ids=[f"p{P.p}-{P.nx}x{P.ny}x{P.nz}{'-conv' if any(P.b) else ''}" for P in CASES])
def test_gmres_sweep_matches_oracle(P, name, method):
    u, f = uniform_pm1(1120 + P.p, 0, P.n_dof), uniform_pm1(1130 + P.p, 0, P.n_dof)
    ref = TierB(P).sweep(u, f, 0.9)
    got, st = sweep(P, method, u, f, 0.9)
    assert st["n_nonconverged"] == 0
    assert st["it_max"] >= 1
    assert rel(got, ref) <= 1e-9


@pytest.mark.parametrize("name,method", METHODS, ids=[m[0] for m in METHODS])
def test_gmres_local_block_solve(name, method):
    """dg_local_block_solve (a8) with GMRES: D_T du = d per cell against dense LU."""
    P = random_problem(5, 4, 2, 3, seed=1140, b=(0.8, 0.3, -0.6), c=True, bc=MIXED)
    d = uniform_pm1(1141, 0, P.n_dof)
    ref = TierB(P).local_solve(d).reshape(-1)
    with dg.DGContext(P) as ctx:
        ctx.set_local_solver(method, 1000)
        du = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.local_block_solve(cuda(d), du, 1e-12)
        st = ctx.stats()
        got = du.cpu().numpy()
    assert st["n_nonconverged"] == 0
    assert rel(got, ref) <= 1e-9


def test_gmres_restarts():
    """Diagonal preconditioner on convection-dominated p = 3 blocks (64 DoF): more than one
    restart cycle of k = 15 steps is needed and the restarted iteration still reaches 1e-12."""
    P = random_problem(4, 3, 3, 3, seed=1150, b=(1.0, 0.7, 0.4), spread=0.0)
    P.K = np.asarray(P.K) * 1e-4
    u, f = uniform_pm1(1151, 0, P.n_dof), uniform_pm1(1152, 0, P.n_dof)
    ref = TierB(P).sweep(u, f, 1.0)
    got, st = sweep(P, dg.DG_LOCAL_GMRES, u, f)
    assert st["n_nonconverged"] == 0
    assert st["it_max"] > 15
    assert rel(got, ref) <= 1e-9


def test_gmres_iteration_cap_flags_cells():
    P = random_problem(4, 3, 3, 3, seed=1160, b=(1.0, 0.7, 0.4), spread=0.0)
    P.K = np.asarray(P.K) * 1e-2
    u, f = uniform_pm1(1161, 0, P.n_dof), uniform_pm1(1162, 0, P.n_dof)
    _, st = sweep(P, dg.DG_LOCAL_GMRES, u, f, max_it=3)
    assert st["n_nonconverged"] > 0
    assert st["it_max"] <= 3


@pytest.mark.parametrize("b", [(1.0, 0.0, 0.0), (1.0, 0.5, 0.3)])
def test_gmres_thomas_convection_dominated(b):
    """eps = 1e-6, |b| ~ 1, h = 1/4 (cell Peclet ~ 2.5e5, the paper's test has 2000): GMRES with
    the tridiagonal preconditioner converges every block and matches the LU sweep."""
    P = random_problem(4, 4, 4, 3, seed=1170, b=b, spread=0.0)
    P.K = np.asarray(P.K) * 1e-6
    u, f = uniform_pm1(1171, 0, P.n_dof), uniform_pm1(1172, 0, P.n_dof)
    ref = TierB(P).sweep(u, f, 1.0)
    got, st = sweep(P, dg.DG_LOCAL_GMRES_THOMAS, u, f)
    assert st["n_nonconverged"] == 0
    assert rel(got, ref) <= 1e-9


@pytest.mark.parametrize("p", [1, 3])
def test_gmres_sor_sweep(p):
    """Red-black SSOR (Alg. 3) with GMRES blocks (the masked colour path)."""
    P = random_problem(6, 3, 3, p, seed=1180 + p, b=(0.7, 0.4, -0.3), c=True, bc=MIXED)
    u, f = uniform_pm1(1181, 0, P.n_dof), uniform_pm1(1182, 0, P.n_dof)
    ref = sor.sor_sweep(TierB(P), u, f, 1.1, symmetric=True)
    with dg.DGContext(P) as ctx:
        ctx.set_local_solver(dg.DG_LOCAL_GMRES, 1000)
        ut = cuda(u)
        ctx.sor_sweep(ut, cuda(f), 1.1, 1e-12, symmetric=True)
        st = ctx.stats()
        got = ut.cpu().numpy()
    assert st["n_nonconverged"] == 0
    assert rel(got, ref) <= 1e-9


def test_gmres_refused_above_p4():
    P = random_problem(2, 2, 2, 5, seed=1190, b=(1.0, 0.0, 0.0))
    with dg.DGContext(P) as ctx:
        with pytest.raises(dg.DGError):
            ctx.set_local_solver(dg.DG_LOCAL_GMRES, 100)
