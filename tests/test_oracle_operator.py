"""Pins for the oracle's operator A (tiers A and B): independent derivations, invariants,
consistency with l_h, and exact reductions. None of these compare the oracle with itself."""
import numpy as np
import pytest

from oracle.kron1d import separable_apply, sipg_1d, to_cell_major
from oracle.tier_a import TierA
from oracle.tier_b import TierB
from synth import DIRICHLET, NEUMANN, Problem, make_config, random_problem

MIXED = (DIRICHLET, NEUMANN, DIRICHLET, DIRICHLET, NEUMANN, DIRICHLET)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("conv", [False, True])
def test_tier_a_equals_tier_b(p, conv):
    """Two independent routes to A_ij = a_h(psi_j, psi_i): brute-force 3D quadrature of
    P:343-357 (tier A) vs 1D quadrature + Kronecker blocks (tier B)."""
    b = (1.0, -0.5, 0.25) if conv else (0.0, 0.0, 0.0)
    P = random_problem(2, 3, 2, p, seed=100 + p, b=b, c=conv, L=(1.0, 0.7, 1.3), bc=MIXED)
    A = TierA(P).assemble()
    B = TierB(P).assemble()
    assert np.abs(A - B).max() <= 1e-13 * np.abs(A).max()


@pytest.mark.parametrize("p", [5, 6, 7])
def test_tier_a_equals_tier_b_high_p(p):
    P = random_problem(1, 1, 2, p, seed=7, b=(0.3, 0.0, -0.2), c=True, L=(1.0, 2.0, 0.5))
    A = TierA(P).assemble()
    B = TierB(P).assemble()
    assert np.abs(A - B).max() <= 1e-13 * np.abs(A).max()


def test_tier_b_per_cell_b_matches_tier_a():
    P = random_problem(2, 2, 2, 2, seed=3, b=(0.2, 0.1, -0.3))
    bc = np.random.default_rng(0).normal(size=(P.n_cells, 3))
    A = TierA(P, b_cells=bc).assemble()
    B = TierB(P, b_cells=bc).assemble()
    assert np.abs(A - B).max() <= 1e-13 * np.abs(A).max()


def test_orientation_invariance():
    """Reading #5: flipping nu_F (and hence which side is '-') changes nothing."""
    P = random_problem(2, 2, 2, 2, seed=5, b=(1.0, 0.5, -0.25), c=True)
    ta = TierA(P)
    A0, A1 = ta.assemble(), ta.assemble(flip=True)
    assert np.abs(A0 - A1).max() <= 1e-14 * np.abs(A0).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_symmetry_and_spd_at_b0(p):
    """SIPG is symmetric for b=0; with a Dirichlet face it is SPD at alpha=1.25
    and alpha=2 (certified by Cholesky), so local CG is well posed."""
    for alpha in (1.25, 2.0):
        P = random_problem(3, 2, 2, p, seed=20 + p, c=False, bc=MIXED, alpha=alpha, spread=1.5)
        A = TierA(P).assemble()
        assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
        np.linalg.cholesky(A)
        tb = TierB(P)
        for c in range(P.n_cells):
            np.linalg.cholesky(tb.diag_block(c))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_constants_annihilated_pure_neumann(p):
    """Pure Neumann, b=0, c=0: A 1 = 0 — the form only sees gradients and jumps."""
    P = random_problem(2, 2, 3, p, seed=30, bc=(NEUMANN,) * 6)
    one = np.ones(P.n_dof)
    for A in (TierA(P).assemble(), TierB(P).assemble()):
        assert np.abs(A @ one).max() <= 1e-12 * np.abs(A).max()
    # ... and the homogeneous-Dirichlet operator does NOT annihilate constants
    P2 = random_problem(2, 2, 3, p, seed=30)
    assert np.abs(TierB(P2).assemble() @ one).max() > 1e-3


def _poly(p, rng):
    """Random u* in Q_p: sum of c_abc x^a y^b z^c, plus its first and second derivatives."""
    C = rng.normal(size=(p + 1, p + 1, p + 1))

    def ev(X, dx=0, dy=0, dz=0):
        x, y, z = X[:, 0], X[:, 1], X[:, 2]
        out = np.zeros(len(X))
        for a in range(p + 1):
            for b in range(p + 1):
                for c in range(p + 1):
                    if a < dx or b < dy or c < dz:
                        continue
                    fa = np.prod(range(a - dx + 1, a + 1)) if dx else 1
                    fb = np.prod(range(b - dy + 1, b + 1)) if dy else 1
                    fc = np.prod(range(c - dz + 1, c + 1)) if dz else 1
                    out += C[a, b, c] * fa * fb * fc * x ** (a - dx) * y ** (b - dy) * z ** (c - dz)
        return out
    return ev


@pytest.mark.parametrize("p", [1, 2, 3])
def test_polynomial_reproduction_inhomogeneous(p):
    """Consistency of a_h with l_h: for any global u* in Q_p, full SPD K, constant
    b and c, mixed Dirichlet (g = u*) / Neumann (j = (b u* - K grad u*).nu) data, the nodal
    interpolant satisfies A I(u*) = l_h exactly. Pins every sign of tier A."""
    rng = np.random.default_rng(p)
    P = Problem(2, 2, 2, p, Lx=1.0, Ly=0.8, Lz=1.2, alpha=1.25, b=(0.7, -0.4, 0.3), bc=MIXED)
    R = rng.normal(size=(3, 3))
    Kf = R @ R.T + 3 * np.eye(3)
    P.K = np.ones(P.n_cells)
    P.c = np.full(P.n_cells, 0.6)
    b = np.array(P.b)
    u = _poly(p, rng)
    E = np.eye(3, dtype=int)

    def grad(X):
        return np.stack([u(X, *E[a]) for a in range(3)], axis=1)

    def f(X):
        lap = sum(Kf[a, bb] * u(X, *(E[a] + E[bb])) for a in range(3) for bb in range(3))
        return -lap + grad(X) @ b + 0.6 * u(X)

    def j(X, nu):
        return (u(X) * (b @ nu)) - grad(X) @ (Kf @ nu)

    ta = TierA(P, K_full=np.tile(Kf, (P.n_cells, 1, 1)))
    A = ta.assemble()
    lh = ta.rhs(f, lambda X: u(X), j)
    uI = ta.interpolate(lambda X: u(X))
    assert rel(A @ uI, lh) < 1e-12


@pytest.mark.parametrize("p", [2, 3, 4])
def test_polynomial_reproduction_homogeneous_tier_b(p):
    """u* = prod_k (x_k/L_k)(1 - x_k/L_k) in Q_2 (the paper's manufactured solution)
    vanishes on the boundary; with K = kappa I, constant b, c = 0, all Dirichlet,
    A I(u*) = M I(f*) with f* = -kappa Lap u* + b.grad u* in Q_2 and M the DG mass matrix
    (tier B with K = 0, b = 0, c = 1)."""
    L = np.array([1.0, 0.8, 1.3])
    kappa = 0.7
    b = np.array([1.0, 0.5, 0.25])
    P = Problem(3, 2, 3, p, Lx=L[0], Ly=L[1], Lz=L[2], alpha=2.0, b=tuple(b))
    P.K = np.full(P.n_cells, kappa)
    Pm = Problem(3, 2, 3, p, Lx=L[0], Ly=L[1], Lz=L[2], alpha=2.0)
    Pm.K = np.zeros(P.n_cells)
    Pm.c = np.ones(P.n_cells)

    def q(X, a):
        t = X[:, a] / L[a]
        return t * (1 - t), (1 - 2 * t) / L[a], -2 / L[a] ** 2

    def ustar(X):
        return q(X, 0)[0] * q(X, 1)[0] * q(X, 2)[0]

    def fstar(X):
        v = [q(X, a) for a in range(3)]
        lap = v[0][2] * v[1][0] * v[2][0] + v[0][0] * v[1][2] * v[2][0] + v[0][0] * v[1][0] * v[2][2]
        gr = [v[0][1] * v[1][0] * v[2][0], v[0][0] * v[1][1] * v[2][0], v[0][0] * v[1][0] * v[2][1]]
        return -kappa * lap + b[0] * gr[0] + b[1] * gr[1] + b[2] * gr[2]

    ta = TierA(P)   # only used for the nodal interpolant (pure geometry)
    uI = ta.interpolate(ustar)
    fI = ta.interpolate(fstar)
    lhs = TierB(P).apply(uI)
    rhs = TierB(Pm).apply(fI)
    assert rel(lhs, rhs) < 1e-12


def test_upwind_direction():
    """K = 0 (degenerate weights, reading #7), c = 0, constant b, u = indicator of one cell T0:
    A u is non-zero only on T0 and its downstream neighbours (b . n_T0 > 0)."""
    P = Problem(3, 3, 3, 2, b=(1.0, -0.5, 0.0))
    P.K = np.zeros(P.n_cells)
    tb = TierB(P)
    c0 = tb.index([1, 1, 1])
    u = np.zeros(P.n_dof)
    u[c0 * P.nd:(c0 + 1) * P.nd] = 1.0
    for A in (tb.assemble(), TierA(P).assemble()):
        out = (A @ u).reshape(P.n_cells, P.nd)
        nz = {c for c in range(P.n_cells) if np.abs(out[c]).max() > 1e-14}
        assert nz == {c0, tb.index([2, 1, 1]), tb.index([1, 0, 1])}


def test_minimal_stencil():
    """A_{T,S} = 0 unless T = S or they share a face."""
    P = random_problem(3, 2, 2, 2, seed=44, b=(0.3, 0.2, 0.1), c=True)
    A = TierA(P).assemble()
    tb = TierB(P)
    nd = P.nd
    for t in range(P.n_cells):
        nbrs = {t} | {nb for nb, _ in tb.nbr_blocks(t)}
        for s in range(P.n_cells):
            blk = A[t * nd:(t + 1) * nd, s * nd:(s + 1) * nd]
            if s in nbrs:
                assert np.abs(blk).max() > 0
            else:
                assert np.abs(blk).max() == 0.0


def test_h_scaling_poisson():
    """K = 1, b = c = 0, cubic cells: A(h) = h A(h=1) (stiffness |T|/h^2, consistency |F|/h and
    penalty gamma |F| all scale like h)."""
    P1 = Problem(3, 3, 3, 2, Lx=3.0, Ly=3.0, Lz=3.0)
    P1.K = np.ones(P1.n_cells)
    P8 = Problem(3, 3, 3, 2, Lx=3 / 8, Ly=3 / 8, Lz=3 / 8)
    P8.K = np.ones(P8.n_cells)
    u = np.random.default_rng(1).uniform(-1, 1, P1.n_dof)
    a1, a8 = TierB(P1).apply(u), TierB(P8).apply(u)
    assert rel(a8, a1 / 8) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3])
def test_quadrature_independence(p):
    """Reading #4: m_o = p+1 Gauss points already integrate every term exactly."""
    P = random_problem(2, 2, 1, p, seed=9, b=(0.5, 0.0, -1.0), c=True)
    for T in (TierA, TierB):
        A3, A1 = T(P).assemble(), T(P, m_o=p + 1).assemble()
        assert np.abs(A3 - A1).max() <= 1e-13 * np.abs(A3).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_kronecker_sum_reduction(p):
    """K = 1, b = c = 0, all Dirichlet: A is the Kronecker sum of independently assembled 1D
    SIPG operators with penalty alpha p(p+2)/h (oracle/kron1d.py)."""
    P = Problem(3, 2, 4, p, Lx=1.0, Ly=0.5, Lz=2.0, alpha=2.0)
    P.K = np.ones(P.n_cells)
    rng = np.random.default_rng(p)
    n = p + 1
    ux, uy, uz = rng.normal(size=P.nx * n), rng.normal(size=P.ny * n), rng.normal(size=P.nz * n)
    u = to_cell_major(P, ux, uy, uz)
    assert rel(TierB(P).apply(u), separable_apply(P, ux, uy, uz)) < 1e-13
    A1, M1 = sipg_1d(4, 2.0, p, 2.0)
    assert np.abs(A1 - A1.T).max() < 1e-12 * np.abs(A1).max()


def _tier_a_parts(P, b_cells=None):
    """The three parts a^v, a^if, a^bf of A assembled separately by tier A's brute-force
    quadrature of P:343-344, P:345-350 and P:352-357 (independent of tier B)."""
    ta = TierA(P, b_cells=b_cells)
    nd, N = P.nd, P.n_cells
    parts = {m: np.zeros((N * nd, N * nd)) for m in (1, 2, 4)}

    def add(m, ct, cr, M):
        parts[m][ct * nd:(ct + 1) * nd, cr * nd:(cr + 1) * nd] += M

    dims = (P.nx, P.ny, P.nz)
    for c in range(N):
        add(1, c, c, ta.volume_block(c))
        co = list(ta.cell_coords(c))
        for axis in range(3):
            if co[axis] + 1 < dims[axis]:
                cu = list(co)
                cu[axis] += 1
                for (ct, cr), M in ta.interior_face_blocks(c, ta.cell_index(*cu), axis).items():
                    add(2, ct, cr, M)
            if co[axis] == 0:
                add(4, c, c, ta.boundary_face_block(c, axis, hi=False))
            if co[axis] == dims[axis] - 1:
                add(4, c, c, ta.boundary_face_block(c, axis, hi=True))
    return parts


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("per_cell_b", [False, True])
def test_apply_parts_match_tier_a_terms(p, per_cell_b):
    """Pins TierB.apply_parts_cells (the reference of the dg_apply_parts GPU tests): each mask
    equals tier A's assembly of that term alone (volume a^v, interior faces a^if, boundary faces
    a^bf), with mixed Dirichlet / Neumann faces, anisotropic K, reaction and b != 0 (constant or
    per cell), and the parts sum to the full apply. A boundary self-term filed under the
    interior mask (or vice versa) fails here."""
    P = random_problem(2, 3, 2, p, seed=60 + p, b=(0.8, -0.4, 0.3), c=True, L=(1.0, 0.7, 1.3),
                       bc=MIXED)
    bc = np.random.default_rng(p).normal(size=(P.n_cells, 3)) if per_cell_b else None
    parts = _tier_a_parts(P, bc)
    tb = TierB(P, b_cells=bc)
    u = np.random.default_rng(10 + p).uniform(-1, 1, P.n_dof)
    cells = range(P.n_cells)
    got = {}
    for mask in (1, 2, 4):
        got[mask] = tb.apply_parts_cells(u, cells, mask).reshape(-1)
        ref = parts[mask] @ u
        assert rel(got[mask], ref) < 1e-13, mask
    for mask in (3, 5, 6, 7):
        combo = tb.apply_parts_cells(u, cells, mask).reshape(-1)
        assert rel(combo, sum(got[m] for m in (1, 2, 4) if mask & m)) < 1e-14
    assert rel(got[1] + got[2] + got[4], tb.apply(u)) < 1e-14
    # the boundary part lives only on cells touching a Dirichlet face
    assert np.abs(got[4].reshape(P.n_cells, P.nd)).max() > 0


def test_problem_per_cell_b_overrides_constant():
    """Problem.b_cells (the data the GPU ABI receives) is what both oracle tiers use."""
    P = random_problem(2, 2, 2, 2, seed=3, b=(0.2, 0.1, -0.3))
    bc = np.random.default_rng(0).normal(size=(P.n_cells, 3))
    A_explicit = TierB(P, b_cells=bc).assemble()
    P.b_cells = bc
    assert np.array_equal(TierB(P).assemble(), A_explicit)
    assert np.abs(TierA(P).assemble() - A_explicit).max() <= 1e-13 * np.abs(A_explicit).max()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_volume_apply_equals_per_cell_volume_blocks(p):
    """TierB.volume_apply (all cells at once, for the large volume-kernel parity cases) equals the
    per-cell a^v blocks, which test_apply_parts_match_tier_a_terms pins to tier A."""
    P = random_problem(3, 2, 2, p, seed=80 + p, b=(0.5, -0.2, 0.1), c=True, L=(1.0, 0.6, 1.4))
    bc = np.random.default_rng(p).normal(size=(P.n_cells, 3))
    tb = TierB(P, b_cells=bc)
    u = np.random.default_rng(p).uniform(-1, 1, P.n_dof)
    ref = tb.apply_parts_cells(u, range(P.n_cells), 1).reshape(-1)
    assert rel(tb.volume_apply(u), ref) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3])
def test_stencil_sub_problem_reproduces_cells(p):
    """Minimal stencil: (A u)_T and the block-Jacobi update of T on a 3 x 3 x 3 problem
    holding T and its face neighbours (tests/stencil_sub.py, the reference of the maximum-size GPU
    parity) equal the full-mesh oracle, on every cell of a mesh with interior, face, edge and
    corner cells."""
    from stencil_sub import gather, sub_problem
    nx, ny, nz = 5, 4, 3
    rng = np.random.default_rng(40 + p)
    K = np.exp(rng.normal(size=nx * ny * nz))
    P = Problem(nx, ny, nz, p, Lx=1.0, Ly=0.7, Lz=1.3, K=K)
    nd = P.nd
    u, f = rng.uniform(-1, 1, P.n_dof), rng.uniform(-1, 1, P.n_dof)
    tb = TierB(P)
    A = tb.apply(u).reshape(-1, nd)
    S = tb.sweep(u, f, 0.9).reshape(-1, nd)
    for cell in range(P.n_cells):
        Ps, gmap, sc = sub_problem(P, K, cell)
        t = TierB(Ps)
        us, fs = gather(u, gmap, nd), gather(f, gmap, nd)
        assert rel(t.apply_cells(us, [sc])[0], A[cell]) < 1e-13
        assert rel(t.sweep_cells(us, fs, 0.9, [sc])[0], S[cell]) < 1e-12
