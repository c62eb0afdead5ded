"""GPU parity of the stored-inverse block-Jacobi smoother (dg_pmf_*): the
assembled D_T against the oracle's Kronecker blocks, the stored inverse against the
oracle's D_T, and the sweep against the oracle's LU sweep (Alg. 2) and the GPU's iterative one."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.tier_b import TierB                                     # noqa: E402
from synth import (DIRICHLET, NEUMANN, make_config, make_vectors,   # noqa: E402
                   random_problem, uniform_pm1)
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


CASES = [random_problem(4, 3, 3, 1, seed=701, c=True, bc=MIXED, spread=1.5),
         random_problem(3, 3, 2, 2, seed=702, bc=MIXED, L=(1.0, 0.6, 1.4)),
         random_problem(3, 2, 2, 3, seed=703, c=True, alpha=1.25),
         random_problem(2, 2, 2, 4, seed=704, bc=MIXED)]
CONV = [random_problem(3, 3, 2, 2, seed=705, b=(1.0, -0.5, 0.25), c=True, bc=MIXED)]


@pytest.mark.parametrize("P", CASES + CONV, ids=[f"p{P.p}{'-conv' if any(P.b) else ''}" for P in CASES + CONV])
def test_assembled_block_matches_oracle(P):
    tb = TierB(P)
    with dg.DGContext(P) as ctx:
        for cell in sorted({0, P.n_cells // 2, P.n_cells - 1}):
            ref = tb.diag_block(cell)
            got = ctx.pmf_block(cell, inverse=False)
            assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("P", CASES, ids=[f"p{P.p}" for P in CASES])
def test_stored_inverse(P):
    tb = TierB(P)
    nd = P.nd
    with dg.DGContext(P) as ctx:
        for cell in sorted({0, P.n_cells - 1}):
            Dinv = ctx.pmf_block(cell, inverse=True)
            assert np.abs(Dinv @ tb.diag_block(cell) - np.eye(nd)).max() <= 1e-11


@pytest.mark.parametrize("P", CASES, ids=[f"p{P.p}" for P in CASES])
def test_pmf_sweep_matches_oracle(P):
    u = uniform_pm1(710 + P.p, 0, P.n_dof)
    f = uniform_pm1(720 + P.p, 0, P.n_dof)
    ref = TierB(P).sweep(u, f, 0.9)
    with dg.DGContext(P) as ctx:
        ctx.pmf_setup()
        ut = cuda(u)
        ctx.pmf_sweep(ut, cuda(f), 0.9)
        torch.cuda.synchronize()
        assert rel(ut.cpu().numpy(), ref) <= 1e-10


def test_pmf_sweep_matches_iterative_sweep_c2():
    """BASELINE configs[1] at full size: the stored-inverse sweep equals the matrix-free sweep
    with local CG to 1e-12 (both exact block solves up to the local tolerance)."""
    P = make_config("C2")
    u, f = make_vectors(P)
    with dg.DGContext(P) as ctx:
        ctx.pmf_setup()
        ft = cuda(f)
        a, b = cuda(u), cuda(u)
        ctx.pmf_sweep(a, ft, 1.0)
        ctx.sweep(b, ft, 1.0, 1e-12)
        torch.cuda.synchronize()
        assert float(torch.linalg.norm(a - b) / torch.linalg.norm(b)) <= 1e-9


def test_pmf_unsupported():
    P = random_problem(2, 2, 2, 5, seed=730)
    with dg.DGContext(P) as ctx:
        with pytest.raises(dg.DGError):
            ctx.pmf_setup()
