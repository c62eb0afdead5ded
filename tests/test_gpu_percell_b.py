"""GPU parity of the round-2 boundary additions against the oracle:

* per-cell advection b_T through the ABI (dg_desc.b_cell; P:290-292 b = b(x)): the volume term
  uses the cell's b, faces b_nu = nu . (b^- + b^+)/2 (DESIGN reading #8), at p = 1..7 for
  dg_apply, D_T, the local solves and the sweep;
* the out-of-place sweep dg_block_jacobi_sweep_to;
* a CG breakdown (non-SPD block) reported as not converged;
* local GMRES at p = 4 and a caller-chosen restart length;
* the stored-inverse smoother with pivoting (b != 0) and across slab boundaries."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.tier_b import TierB                                    # noqa: E402
from synth import DIRICHLET, NEUMANN, random_problem, uniform_pm1  # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

APPLY_TOL = 1e-12
SWEEP_TOL = 1e-9
MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def vec(P, seed):
    return uniform_pm1(seed, 0, P.n_dof), uniform_pm1(seed + 1, 0, P.n_dof)


SIZES = {1: (9, 7, 5), 2: (7, 5, 4), 3: (5, 4, 3), 4: (4, 3, 3), 5: (3, 3, 2), 6: (3, 2, 2), 7: (3, 2, 1)}


def bfield_problem(p, seed=800, scale=1.0):
    nx, ny, nz = SIZES[p]
    P = random_problem(nx, ny, nz, p, seed=seed + p, spread=1.0, b=(0.3, 0.1, -0.2), c=True,
                       bc=MIXED, L=(1.0, 0.7, 1.3))
    P.b_cells = scale * np.random.default_rng(seed + p).normal(size=(P.n_cells, 3))
    P.local_solver = "bicgstab"
    return P


@pytest.mark.parametrize("p", range(1, 8))
def test_per_cell_b_apply_and_block_diag(p):
    P = bfield_problem(p)
    u, _ = vec(P, 60)
    tb = TierB(P)
    with dg.DGContext(P) as ctx:
        ut = cuda(u)
        out = torch.empty_like(ut)
        ctx.apply(ut, out)
        assert rel(host(out), tb.apply(u)) <= APPLY_TOL
        for mask in (1, 2, 4):
            ctx.apply_parts(ut, out, mask)
            assert rel(host(out), tb.apply_parts_cells(u, range(P.n_cells), mask).reshape(-1)) <= APPLY_TOL
        ctx.block_diag_apply(ut, out)
        assert rel(host(out), tb.block_diag_apply(u).reshape(-1)) <= APPLY_TOL


@pytest.mark.parametrize("p", range(1, 8))
def test_per_cell_b_local_solve_and_sweep(p):
    P = bfield_problem(p)
    d, f = vec(P, 61)
    tb = TierB(P)
    ref = tb.local_solve(d)
    with dg.DGContext(P) as ctx:
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.local_block_solve(cuda(d), out, 1e-12)
        got = host(out).reshape(P.n_cells, P.nd)
        assert ctx.stats()["n_nonconverged"] == 0
        for c in range(P.n_cells):
            assert rel(got[c], ref[c]) <= 1e-10, c
        ut = cuda(d)
        ctx.sweep(ut, cuda(f), 0.8, 1e-12)
        assert rel(host(ut), tb.sweep(d, f, 0.8)) <= SWEEP_TOL


def test_per_cell_b_constant_field_equals_constant_b():
    """b_cell filled with the constant b reproduces the constant-b operator bit for bit
    (the face mean (b + b)/2 = b is exact)."""
    P = random_problem(5, 4, 3, 3, seed=9, b=(0.7, -0.4, 0.3), c=True)
    u, _ = vec(P, 62)
    with dg.DGContext(P) as ctx:
        a = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.apply(cuda(u), a)
        a = host(a)
    P.b_cells = np.tile(np.asarray(P.b), (P.n_cells, 1))
    with dg.DGContext(P) as ctx:
        b = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.apply(cuda(u), b)
        b = host(b)
    assert rel(b, a) <= 1e-15


def test_per_cell_b_partition_invariance():
    """z-slabs with the per-cell b field: the slab-boundary faces average the ghost layer's b."""
    P = bfield_problem(2, seed=810)
    P = random_problem(4, 3, 6, 2, seed=811, spread=1.0, c=True)
    P.b_cells = np.random.default_rng(3).normal(size=(P.n_cells, 3))
    u, f = vec(P, 63)
    with dg.DGContext(P) as one:
        ut = cuda(u)
        ref_A = torch.empty_like(ut)
        one.apply(ut, ref_A)
        one.sweep(ut, cuda(f), 0.9, 1e-12)
        ref_A, ref_S = host(ref_A), host(ut)
    nd, nxy, G = P.nd, P.nx * P.ny, 2
    ctxs = [dg.DGContext(P, rank=r, nranks=G, halo_mode=dg.DG_HALO_EXTERNAL) for r in range(G)]
    try:
        parts_u = [cuda(u[c.cell_begin * nd:c.cell_end * nd]) for c in ctxs]
        parts_f = [cuda(f[c.cell_begin * nd:c.cell_end * nd]) for c in ctxs]
        for r, c in enumerate(ctxs):
            c.fill_ghosts(parts_u[r - 1][-nxy * nd:] if r > 0 else None,
                          parts_u[r + 1][:nxy * nd] if r < G - 1 else None)
        outs = []
        for r, c in enumerate(ctxs):
            o = torch.empty_like(parts_u[r])
            c.apply(parts_u[r], o)
            outs.append(host(o))
        assert np.array_equal(np.concatenate(outs), ref_A)
        for r, c in enumerate(ctxs):
            c.sweep(parts_u[r], parts_f[r], 0.9, 1e-12)
        assert np.array_equal(np.concatenate([host(x) for x in parts_u]), ref_S)
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_sweep_to_equals_in_place_sweep(p):
    nx, ny, nz = SIZES[p]
    P = random_problem(nx, ny, nz, p, seed=820 + p, spread=1.0)
    u, f = vec(P, 64)
    with dg.DGContext(P) as ctx:
        ut, ft = cuda(u), cuda(f)
        un = torch.empty_like(ut)
        ctx.sweep_to(ut, ft, un, 0.9, 1e-12)
        assert np.array_equal(host(ut), u)          # u is read only
        ctx.sweep(ut, ft, 0.9, 1e-12)
        assert np.array_equal(host(un), host(ut))
        with pytest.raises(dg.DGError):
            ctx.sweep_to(ut, ft, ut, 0.9, 1e-12)


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_cg_breakdown_reported_not_converged(p):
    """CG forced on strongly convective (nonsymmetric, indefinite-for-CG) blocks: every cell that
    stops on p^T D_T p <= 0 or the cap is counted as not converged, never as converged with a
    wrong answer: any cell the stats call converged satisfies the tolerance."""
    nx, ny, nz = SIZES[p]
    P = random_problem(nx, ny, nz, p, seed=830 + p, spread=0.5, b=(40.0, -30.0, 25.0))
    P.K = np.full(P.n_cells, 1e-3)
    d, _ = vec(P, 65)
    tb = TierB(P)
    with dg.DGContext(P) as ctx:
        ctx.set_local_solver(dg.DG_LOCAL_CG, 60)
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.local_block_solve(cuda(d), out, 1e-12)
        got = host(out).reshape(P.n_cells, P.nd)
        st = ctx.stats()
    assert st["n_nonconverged"] > 0
    D = d.reshape(P.n_cells, P.nd)
    n_ok = 0
    for c in range(P.n_cells):
        res = np.linalg.norm(D[c] - tb.diag_block(c) @ got[c]) / np.linalg.norm(D[c])
        n_ok += res <= 1e-10
    assert n_ok >= P.n_cells - st["n_nonconverged"]


@pytest.mark.parametrize("method", [dg.DG_LOCAL_GMRES, dg.DG_LOCAL_GMRES_THOMAS], ids=["gmres", "gmres-thomas"])
def test_gmres_p4(method):
    """Local GMRES at p = 4 (the paper's convection test runs GMRES at p = 2, 3, 4; P:1167-1169,
    Table 6): 9 basis vectors in tensor memory."""
    P = random_problem(4, 3, 3, 4, seed=840, spread=0.5, b=(1.0, -0.5, 0.25), c=True, bc=MIXED)
    d, f = vec(P, 66)
    tb = TierB(P)
    ref = tb.local_solve(d)
    with dg.DGContext(P) as ctx:
        ctx.set_local_solver(method, 2000)
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.local_block_solve(cuda(d), out, 1e-12)
        got = host(out).reshape(P.n_cells, P.nd)
        assert ctx.stats()["n_nonconverged"] == 0
        for c in range(P.n_cells):
            assert rel(got[c], ref[c]) <= 1e-10
        ut = cuda(d)
        ctx.sweep(ut, cuda(f), 1.0, 1e-12)
        assert rel(host(ut), tb.sweep(d, f, 1.0)) <= SWEEP_TOL


@pytest.mark.parametrize("k", [3, 6])
def test_gmres_restart_length(k):
    """A shorter restart converges to the same solves with more Arnoldi steps."""
    P = random_problem(4, 4, 3, 3, seed=850, spread=0.5, b=(1.0, -0.5, 0.25))
    d, _ = vec(P, 67)
    ref = TierB(P).local_solve(d)
    with dg.DGContext(P) as ctx:
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        its = []
        for kr in (0, k):
            ctx.set_local_solver(dg.DG_LOCAL_GMRES, 3000, kr)
            ctx.local_block_solve(cuda(d), out, 1e-12)
            st = ctx.stats()
            assert st["n_nonconverged"] == 0
            got = host(out).reshape(P.n_cells, P.nd)
            for c in range(P.n_cells):
                assert rel(got[c], ref[c]) <= 1e-10
            its.append(st["it_sum"])
    assert its[1] >= its[0]


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_pmf_convective_blocks_with_pivoting(p):
    nx, ny, nz = SIZES[p]
    P = random_problem(nx, ny, nz, p, seed=860 + p, spread=1.0, b=(2.0, -1.0, 0.5), c=True, bc=MIXED)
    P.b_cells = np.random.default_rng(p).normal(size=(P.n_cells, 3)) * 2.0
    u, f = vec(P, 68)
    tb = TierB(P)
    with dg.DGContext(P) as ctx:
        ctx.pmf_setup()
        for c in (0, P.n_cells - 1):
            D = tb.diag_block(c)
            assert rel(ctx.pmf_block(c, inverse=False), D) <= 1e-13
            assert rel(ctx.pmf_block(c, inverse=True), np.linalg.inv(D)) <= 1e-10
        ut = cuda(u)
        ctx.pmf_sweep(ut, cuda(f), 0.9)
        assert rel(host(ut), tb.sweep(u, f, 0.9)) <= 1e-10


def test_pmf_partition_invariance():
    """Stored inverses across z-slabs: the slab-boundary faces of D_T are interior faces whose
    neighbour coefficients come from the ghost layer (bit-for-bit equal to one slab)."""
    P = random_problem(4, 3, 6, 2, seed=870, spread=1.5, c=True)
    u, f = vec(P, 69)
    with dg.DGContext(P) as one:
        one.pmf_setup()
        ut = cuda(u)
        one.pmf_sweep(ut, cuda(f), 0.9)
        ref = host(ut)
    nd, nxy, G = P.nd, P.nx * P.ny, 2
    ctxs = [dg.DGContext(P, rank=r, nranks=G, halo_mode=dg.DG_HALO_EXTERNAL) for r in range(G)]
    try:
        parts_u = [cuda(u[c.cell_begin * nd:c.cell_end * nd]) for c in ctxs]
        parts_f = [cuda(f[c.cell_begin * nd:c.cell_end * nd]) for c in ctxs]
        for r, c in enumerate(ctxs):
            c.pmf_setup()
            c.fill_ghosts(parts_u[r - 1][-nxy * nd:] if r > 0 else None,
                          parts_u[r + 1][:nxy * nd] if r < G - 1 else None)
        torch.cuda.synchronize()
        for r, c in enumerate(ctxs):
            c.pmf_sweep(parts_u[r], parts_f[r], 0.9)
        got = np.concatenate([host(x) for x in parts_u])
    finally:
        for c in ctxs:
            c.close()
    assert np.array_equal(got, ref)
