"""GPU parity of the red-black block SOR / SSOR sweep (dg_block_sor_sweep, Alg. 3; SURVEY 8(f)
NEXT-2) against the oracle (oracle/sor.py, exact LU local solves). Bar: relative L2 <= 1e-9, the
sweep tolerance of BASELINE.json, local solves to 1e-12; p = 1..7, CG and BiCGStab blocks."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import sor                                              # noqa: E402
from oracle.tier_b import TierB                                     # noqa: E402
from synth import DIRICHLET, NEUMANN, random_problem, uniform_pm1   # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


CASES = []
for p in range(1, 8):
    nx, ny, nz = {1: (7, 5, 4), 2: (5, 4, 3), 3: (5, 3, 3), 4: (4, 3, 2), 5: (3, 3, 2),
                  6: (3, 2, 2), 7: (3, 2, 1)}[p]
    CASES.append((random_problem(nx, ny, nz, p, seed=600 + p, spread=1.2), p % 2 == 0, 1.0))
    if p <= 4:
        CASES.append((random_problem(nx, ny, nz, p, seed=610 + p, b=(1.0, -0.5, 0.25), c=True,
                                     bc=MIXED, L=(1.0, 0.6, 1.4)), p % 2 == 1, 1.2))


# even nx: p <= 3 runs the compact colour map (in-place half-sweeps over one colour's cells)
for p, shape in ((1, (8, 5, 3)), (2, (6, 4, 3)), (3, (4, 3, 5))):
    CASES.append((random_problem(*shape, p, seed=650 + p, spread=1.0), True, 1.1))
    CASES.append((random_problem(*shape, p, seed=660 + p, b=(0.7, 0.4, -0.3), c=True, bc=MIXED), False, 0.9))


@pytest.mark.parametrize("P,symmetric,omega", CASES,
                         ids=[f"p{c[0].p}-nx{c[0].nx}-{'conv' if any(c[0].b) else 'diff'}-{'ssor' if c[1] else 'sor'}"
                              for c in CASES])
def test_sor_matches_oracle(P, symmetric, omega):
    u = uniform_pm1(620 + P.p, 0, P.n_dof)
    f = uniform_pm1(630 + P.p, 0, P.n_dof)
    ref = sor.sor_sweep(TierB(P), u, f, omega, symmetric=symmetric)
    with dg.DGContext(P) as ctx:
        ut = cuda(u)
        ctx.sor_sweep(ut, cuda(f), omega, 1e-12, symmetric=symmetric)
        torch.cuda.synchronize()
        got = ut.cpu().numpy()
        st = ctx.stats()
    assert st["n_nonconverged"] == 0
    assert rel(got, ref) <= 1e-9


def test_gauss_seidel_beats_jacobi_on_gpu():
    """Poisson, omega = 1, zero initial guess: after the same number of sweeps the red-black
    block Gauss-Seidel residual is below the block-Jacobi one (2-cyclic ordering)."""
    P = random_problem(6, 5, 4, 2, seed=640, aniso=False, spread=0.0)
    f = cuda(uniform_pm1(641, 0, P.n_dof))
    with dg.DGContext(P) as ctx:
        uj = torch.zeros_like(f)
        ug = torch.zeros_like(f)
        for _ in range(4):
            ctx.sweep(uj, f, 1.0, 1e-12)
            ctx.sor_sweep(ug, f, 1.0, 1e-12)
        rj, rg = torch.empty_like(f), torch.empty_like(f)
        ctx.apply(uj, rj)
        ctx.apply(ug, rg)
        nj = float(torch.linalg.norm(f - rj))
        ng = float(torch.linalg.norm(f - rg))
    assert ng < 0.8 * nj
