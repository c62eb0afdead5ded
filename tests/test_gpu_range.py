"""GPU checks of the z-layer range calls (dg_apply_range, dg_block_jacobi_sweep_range; include/dg.h):
the chunks of a slab, in any order, reproduce dg_apply / dg_block_jacobi_sweep_to bit for bit
(the rows of A u, and of the out-of-place sweep, Alg. 2, are per cell), a
range call writes only its own cells, and misaligned or multi-slab ranges are refused. The full
calls themselves are pinned to the oracle in test_gpu_parity.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from synth import DIRICHLET, NEUMANN, random_problem, uniform_pm1  # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)
# meshes with several granules of z-layers per degree (nx * ny a multiple of the group sizes)
MESH = {1: (8, 8, 7), 2: (8, 5, 9), 3: (8, 4, 7), 4: (6, 4, 6), 5: (4, 3, 5), 6: (3, 4, 5), 7: (2, 3, 4)}


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def chunks(nz, g, seed):
    """Consecutive z-ranges of g layers (the last one may be shorter), in a seeded random order."""
    bounds = list(range(0, nz, g)) + [nz]
    rs = [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]
    np.random.default_rng(seed).shuffle(rs)
    return rs


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("kind", ["poisson", "conv"])
def test_range_calls_equal_full_calls_bitwise(p, kind):
    nx, ny, nz = MESH[p]
    if kind == "poisson":
        P = random_problem(nx, ny, nz, p, seed=700 + p, spread=1.0)
    else:
        P = random_problem(nx, ny, nz, p, seed=710 + p, b=(1.0, -0.5, 0.25), c=True, bc=MIXED,
                           L=(1.0, 0.7, 1.3))
    u, f = uniform_pm1(720 + p, 0, P.n_dof), uniform_pm1(730 + p, 0, P.n_dof)
    with dg.DGContext(P) as ctx:
        g = ctx.range_granule()
        assert g >= 1
        ut, ft = cuda(u), cuda(f)
        full = torch.empty_like(ut)
        ctx.apply(ut, full)
        part = torch.full_like(ut, float("nan"))
        for zb, ze in chunks(nz, g, p):
            ctx.apply_range(ut, part, zb, ze)
        torch.cuda.synchronize()
        assert torch.equal(part, full)
        # sweeps (local tolerance 1e-12) and the per-cell iteration statistics
        ref = torch.empty_like(ut)
        ctx.sweep_to(ut, ft, ref, 0.9, 1e-12)
        st_full = ctx.stats()
        got = torch.full_like(ut, float("nan"))
        for zb, ze in chunks(nz, g, 100 + p):
            ctx.sweep_range_to(ut, ft, got, zb, ze, 0.9, 1e-12)
        st_part = ctx.stats()
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        assert st_part["it_sum"] == st_full["it_sum"] and st_part["it_max"] == st_full["it_max"]


@pytest.mark.parametrize("p", [2, 4, 6])
def test_range_writes_only_its_cells(p):
    nx, ny, nz = MESH[p]
    P = random_problem(nx, ny, nz, p, seed=740 + p)
    u, f = uniform_pm1(750 + p, 0, P.n_dof), uniform_pm1(760 + p, 0, P.n_dof)
    nd = (p + 1) ** 3
    with dg.DGContext(P) as ctx:
        g = ctx.range_granule()
        zb, ze = g, min(nz, 2 * g)
        lo, hi = zb * nx * ny * nd, ze * nx * ny * nd
        ut, ft = cuda(u), cuda(f)
        for call in ("apply", "sweep"):
            out = torch.full_like(ut, float("nan"))
            if call == "apply":
                ctx.apply_range(ut, out, zb, ze)
            else:
                ctx.sweep_range_to(ut, ft, out, zb, ze)
            o = out.cpu().numpy()
            assert np.isnan(o[:lo]).all() and np.isnan(o[hi:]).all()
            assert np.isfinite(o[lo:hi]).all()
        # an empty range is a no-op
        out = torch.full_like(ut, float("nan"))
        ctx.apply_range(ut, out, zb, zb)
        assert torch.isnan(out).all()


def test_range_bounds_refused():
    # p = 2: plane groups of 40 cells and line groups of 32 -> 160 cells; nx * ny = 20: 8 layers
    P = random_problem(5, 4, 17, 2, seed=770)
    u = uniform_pm1(771, 0, P.n_dof)
    with dg.DGContext(P) as ctx:
        g = ctx.range_granule()
        assert g == 8
        ut = cuda(u)
        out = torch.empty_like(ut)
        ctx.apply_range(ut, out, 8, 16)
        ctx.apply_range(ut, out, 16, 17)          # the last layer may end a range
        for zb, ze in [(1, 8), (0, 5), (8, 18), (-8, 0), (16, 8)]:
            with pytest.raises(dg.DGError):
                ctx.apply_range(ut, out, zb, ze)
            with pytest.raises(dg.DGError):
                ctx.sweep_range_to(ut, ut.clone(), out, zb, ze)
        with pytest.raises(dg.DGError):
            ctx.apply_range(ut, ut, 0, 8)         # aliasing


def test_range_refused_for_slabs():
    P = random_problem(4, 4, 6, 3, seed=780)
    with dg.DGContext(P, rank=0, nranks=2, halo_mode=dg.DG_HALO_EXTERNAL) as ctx:
        n = ctx.n_local_dof
        a = torch.zeros(n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        with pytest.raises(dg.DGError):
            ctx.apply_range(a, b, 0, 1)
