"""GPU parity of every kernel variant whose speed is reported or selectable (dg_set_kernel_variant),
and of the persistent volume kernels on meshes with more cell groups than resident CTA slots (the
next-group prefetch loop), every DoF against the oracle.

Tolerances (BASELINE.json north_star): relative L2 <= 1e-12 for dg_apply and its parts, <= 1e-9
after a sweep; local solves vs dense LU <= 1e-10 per cell."""
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


# ---- persistent volume kernels, multi-wave ------------------------------------------------
# more cell groups than the resident CTA slots (148 SMs x 16 CTAs at p <= 4) (an upper bound for every k_volume*): each
# CTA walks several groups, so the register / cp.async prefetch of the next group runs
# (p = 5, 6, 7: the lean line kernel k_volume_line; with -DDG_PLANE_VOL67=1 the plane-per-lane k_volume_s)
MULTIWAVE = {1: (47, 43, 38), 2: (41, 37, 31), 3: (44, 43, 41), 4: (31, 30, 31), 5: (21, 19, 17),
             6: (19, 17, 16), 7: (15, 13, 12)}


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("variant", [0, dg.DG_VARIANT_VOLUME_PREFETCH], ids=["default", "prefetch"])
@pytest.mark.parametrize("gen", [False, True], ids=["diffusion", "conv-reaction"])
def test_volume_kernel_multiwave_every_dof(p, variant, gen):
    if variant and p != 3:
        pytest.skip("the prefetch variant differs from the default at p = 3 only")
    nx, ny, nz = MULTIWAVE[p]
    P = random_problem(nx, ny, nz, p, seed=400 + p, spread=1.0, b=(0.6, -0.3, 0.2) if gen else (0, 0, 0),
                       c=gen, L=(1.0, 0.8, 1.2))
    if gen:
        P.b_cells = np.random.default_rng(p).normal(size=(P.n_cells, 3))
    u, _ = vec(P, 40 + p)
    ref = TierB(P).volume_apply(u)
    with dg.DGContext(P) as ctx:
        ctx.set_kernel_variant(variant)
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.apply_parts(cuda(u), out, dg.MASK_VOLUME)
        got = host(out)
    assert rel(got, ref) <= APPLY_TOL


# ---- the line family at p <= 4 (DG_VARIANT_LINE) ---------------------------------------------
def small_problems():
    out = []
    for p in range(1, 5):
        nx, ny, nz = {1: (9, 7, 5), 2: (7, 5, 4), 3: (5, 4, 3), 4: (4, 3, 3)}[p]
        out.append(("poisson", random_problem(nx, ny, nz, p, seed=500 + p, spread=1.5)))
        out.append(("conv", random_problem(nx, ny, nz, p, seed=600 + p, b=(1.0, -0.5, 0.25), c=True,
                                           bc=MIXED, L=(1.0, 0.6, 1.4))))
    return out


SMALL = small_problems()
SMALL_IDS = [f"{k}-p{P.p}" for k, P in SMALL]


@pytest.mark.parametrize("kind,P", SMALL, ids=SMALL_IDS)
def test_line_family_apply_parts_diag(kind, P):
    u, _ = vec(P, 50)
    tb = TierB(P)
    with dg.DGContext(P) as ctx:
        ctx.set_kernel_variant(dg.DG_VARIANT_LINE)
        ut = cuda(u)
        out = torch.empty_like(ut)
        ctx.apply(ut, out)
        assert rel(host(out), tb.apply(u)) <= APPLY_TOL
        for mask in (1, 2, 4):
            ctx.apply_parts(ut, out, mask)
            ref = tb.apply_parts_cells(u, range(P.n_cells), mask).reshape(-1)
            if np.linalg.norm(ref) > 0:
                assert rel(host(out), ref) <= APPLY_TOL, mask
        ctx.block_diag_apply(ut, out)
        assert rel(host(out), tb.block_diag_apply(u).reshape(-1)) <= APPLY_TOL


@pytest.mark.parametrize("kind,P", SMALL, ids=SMALL_IDS)
def test_line_family_local_solve_and_sweep(kind, P):
    d, f = vec(P, 51)
    tb = TierB(P)
    ref_solve = tb.local_solve(d)
    ref_sweep = tb.sweep(d, f, 0.8)
    with dg.DGContext(P) as ctx:
        ctx.set_kernel_variant(dg.DG_VARIANT_LINE)
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.local_block_solve(cuda(d), out, 1e-12)
        got = host(out).reshape(P.n_cells, P.nd)
        assert ctx.stats()["n_nonconverged"] == 0
        for c in range(P.n_cells):
            assert rel(got[c], ref_solve[c]) <= 1e-10
        ut = cuda(d)
        ctx.sweep(ut, cuda(f), 0.8, 1e-12)
        assert rel(host(ut), ref_sweep) <= SWEEP_TOL


# ---- BiCGStab without tensor memory (p = 3), CTA-barrier line solvers (p = 4..6) -------------
def _sweep_case(P, variant, method=dg.DG_LOCAL_AUTO, seed=52):
    u, f = vec(P, seed)
    ref = TierB(P).sweep(u, f, 0.9)
    with dg.DGContext(P) as ctx:
        ctx.set_kernel_variant(variant)
        ctx.set_local_solver(method, 1000)
        ut = cuda(u)
        ctx.sweep(ut, cuda(f), 0.9, 1e-12)
        got = host(ut)
        assert ctx.stats()["n_nonconverged"] == 0
    assert rel(got, ref) <= SWEEP_TOL


def test_bicgstab_shared_memory_variant_p3():
    P = random_problem(5, 4, 3, 3, seed=700, b=(1.0, -0.5, 0.25), c=True, bc=MIXED)
    _sweep_case(P, dg.DG_VARIANT_NO_TMEM)


@pytest.mark.parametrize("p", [4, 5, 6])
@pytest.mark.parametrize("conv", [False, True], ids=["cg", "bicgstab"])
def test_line_cta_solvers(p, conv):
    nx, ny, nz = {4: (4, 3, 3), 5: (3, 3, 2), 6: (3, 2, 2)}[p]
    P = random_problem(nx, ny, nz, p, seed=710 + p, spread=1.0,
                       b=(0.8, -0.3, 0.2) if conv else (0.0, 0.0, 0.0), c=conv)
    _sweep_case(P, dg.DG_VARIANT_LINE_CG_CTA)


def test_unknown_variant_rejected():
    P = random_problem(2, 2, 2, 2, seed=1)
    with dg.DGContext(P) as ctx:
        with pytest.raises(dg.DGError):
            ctx.set_kernel_variant(1 << 8)


# ---- the warp-mode nodal D_T at p = 4 (k_dt_warps): ragged last CTA, slab-free and both term sets
@pytest.mark.parametrize("gen", [False, True], ids=["diffusion", "conv-reaction"])
@pytest.mark.parametrize("mesh", [(5, 3, 3), (7, 5, 3)], ids=["45cells", "105cells"])
def test_block_diag_warp_kernel_p4_every_dof(gen, mesh):
    P = random_problem(*mesh, 4, seed=510, spread=1.5, b=(0.7, -0.4, 0.3) if gen else (0, 0, 0),
                       c=gen, bc=MIXED if gen else (DIRICHLET,) * 6, L=(1.0, 0.7, 1.3))
    if gen:
        P.b_cells = np.random.default_rng(5).normal(size=(P.n_cells, 3))
    u, _ = vec(P, 61)
    ref = TierB(P).block_diag_apply(u).reshape(-1)
    for variant in (0, dg.DG_VARIANT_LINE):
        with dg.DGContext(P) as ctx:
            ctx.set_kernel_variant(variant)
            out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
            ctx.block_diag_apply(cuda(u), out)
            got = host(out)
        assert rel(got, ref) <= APPLY_TOL, variant


# ---- dg_apply at p = 4: the mass-folded kernel (default) and the face-array warp kernel ------
@pytest.mark.parametrize("variant", [0, dg.DG_VARIANT_APPLY_NOFOLD], ids=["fold", "face-arrays"])
@pytest.mark.parametrize("gen", [False, True], ids=["diffusion", "conv-reaction"])
@pytest.mark.parametrize("mesh", [(5, 3, 3), (7, 5, 3)], ids=["45cells", "105cells"])
def test_apply_p4_kernels_every_dof(variant, gen, mesh):
    """Both p = 4 apply kernels on meshes with a ragged last CTA (4 cells per CTA), mixed
    Dirichlet / Neumann faces, anisotropic cells and K; every DoF against the oracle, and the two
    kernels against each other."""
    nx, ny, nz = mesh
    P = random_problem(nx, ny, nz, 4, seed=760 + nx, spread=1.5, bc=MIXED, L=(1.0, 0.6, 1.4),
                       b=(0.7, -0.4, 0.3) if gen else (0.0, 0.0, 0.0), c=gen)
    if gen:
        P.b_cells = np.random.default_rng(nx).normal(size=(P.n_cells, 3))
    u, _ = vec(P, 61)
    ref = TierB(P).apply(u)
    with dg.DGContext(P) as ctx:
        ctx.set_kernel_variant(variant)
        out = torch.empty(P.n_dof, dtype=torch.float64, device="cuda")
        ctx.apply(cuda(u), out)
        got = host(out)
    assert rel(got, ref) <= 1e-12
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()
