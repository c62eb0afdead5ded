"""Maximum sizes: one slab with more than 2^31 DoF (17.7 GB per vector), so that every cell
offset, DoF count and byte offset that would wrap in 32 bits is exercised in the bench's launch
configuration (dg_apply, and one block-Jacobi sweep with the local CG to 1e-12).

The oracle cannot hold such a vector, and does not have to: (A u)_T and the sweep's update of T
depend on u in T and its six face neighbours, on K of those cells, on h and on which faces of T
lie on the boundary (minimal stencil). Each sampled cell is therefore checked against
the oracle on a 3 x 3 x 3 mesh of the same cell size that holds T (at the centre, or on the
matching boundary side) with the neighbours' K and u read back from the device vector."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle.tier_b import TierB                                    # noqa: E402
from synth import Problem, normal, uniform_pm1                      # noqa: E402
import paper_1805_11930_b200 as dg                                  # noqa: E402
from stencil_sub import gather, sub_problem                        # noqa: E402

APPLY_TOL = 1e-12
SWEEP_TOL = 1e-9
BLOCK = (1 << 24) + 3          # seeded block length, coprime with the cell size


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def tiled(seed, n_dof):
    """A seeded U[-1, 1) block repeated over the device vector (generated once on the host; the
    period is not a multiple of the cell size, so no two neighbouring cells hold equal data)."""
    blk = torch.from_numpy(uniform_pm1(seed, 0, BLOCK)).cuda()
    out = torch.empty(n_dof, dtype=torch.float64, device="cuda")
    for s in range(0, n_dof, BLOCK):
        m = min(BLOCK, n_dof - s)
        out[s:s + m] = blk[:m]
    return out


@pytest.mark.parametrize("p,mesh", [(7, (128, 128, 264)), (4, (160, 160, 170))],
                         ids=["Q7-2.2e9dof", "Q4-5.4e8dof"])
def test_more_than_2_31_dof(p, mesh):
    nx, ny, nz = mesh
    N = nx * ny * nz
    nd = (p + 1) ** 3
    n_dof = N * nd
    need = 4 * n_dof * 8 + (4 << 30)
    free, _ = torch.cuda.mem_get_info()
    if free < need:
        pytest.skip(f"needs {need >> 30} GiB of device memory")
    assert n_dof * 8 > 2 ** 32 and (p != 7 or n_dof > 2 ** 31)
    K = np.exp(normal(911, 0, N))
    P = Problem(nx, ny, nz, p, K=K)
    u = tiled(912, n_dof)
    f = tiled(913, n_dof)
    Au = torch.empty_like(u)
    un = torch.empty_like(u)
    rng = np.random.default_rng(5)
    cells = sorted({0, nx - 1, N - 1, N - nx, N - nx * ny, nx * ny * (nz // 2) + nx * (ny // 2) + nx // 2}
                   | set(rng.integers(N - N // 8, N, 3).tolist()) | set(rng.integers(0, N, 3).tolist()))
    with dg.DGContext(P) as ctx:
        ctx.apply(u, Au)
        ctx.sweep_to(u, f, un, 1.0, 1e-12)
        torch.cuda.synchronize()
        st = ctx.stats()
    assert st["n_cells"] == N and st["n_nonconverged"] == 0
    assert bool(torch.isfinite(Au).all()) and bool(torch.isfinite(un).all())
    for cell in cells:
        Ps, gmap, sc = sub_problem(P, K, cell)
        tb = TierB(Ps)
        us, fs = gather(u, gmap, nd), gather(f, gmap, nd)
        ref_a = tb.apply_cells(us, [sc])[0]
        got_a = Au[cell * nd:(cell + 1) * nd].cpu().numpy()
        assert rel(got_a, ref_a) <= APPLY_TOL, (cell, rel(got_a, ref_a))
        ref_s = tb.sweep_cells(us, fs, 1.0, [sc])[0]
        got_s = un[cell * nd:(cell + 1) * nd].cpu().numpy()
        assert rel(got_s, ref_s) <= SWEEP_TOL, (cell, rel(got_s, ref_s))
    del u, f, Au, un
    torch.cuda.empty_cache()
