"""Test helper (no arithmetic of the method): the 3 x 3 x 3 problem that holds one cell T of a large
mesh with its face neighbours, for checking single cells of vectors the oracle cannot hold.
(A u)_T and the block-Jacobi update of T depend on u and K in T and its six face neighbours, on h
and on which faces of T are boundary faces (minimal stencil); pinned on every cell of
a small mesh in tests/test_oracle_operator.py::test_stencil_sub_problem_reproduces_cells."""
import numpy as np

from synth import Problem


def sub_problem(P, K, cell):
    """The 3 x 3 x 3 problem around `cell` and the map sub-cell -> global cell (or -1)."""
    dims = (P.nx, P.ny, P.nz)
    co = (cell % P.nx, (cell // P.nx) % P.ny, cell // (P.nx * P.ny))
    # position of T in the sub-mesh: on the boundary side it touches, else the centre
    so = [0 if co[d] == 0 else (2 if co[d] == dims[d] - 1 else 1) for d in range(3)]
    h = P.h
    Ks = np.ones(27)
    gmap = -np.ones(27, dtype=np.int64)
    for sz in range(3):
        for sy in range(3):
            for sx in range(3):
                g = [co[0] + sx - so[0], co[1] + sy - so[1], co[2] + sz - so[2]]
                if all(0 <= g[d] < dims[d] for d in range(3)):
                    gc = g[0] + P.nx * (g[1] + P.ny * g[2])
                    gmap[sx + 3 * (sy + 3 * sz)] = gc
                    Ks[sx + 3 * (sy + 3 * sz)] = K[gc]
    Ps = Problem(3, 3, 3, P.p, Lx=3 * h[0], Ly=3 * h[1], Lz=3 * h[2], alpha=P.alpha, K=Ks)
    return Ps, gmap, so[0] + 3 * (so[1] + 3 * so[2])


def gather(t, gmap, nd):
    """The sub-mesh vector: the device vector's cells where they exist (T and its face
    neighbours are the ones that matter), zero elsewhere."""
    out = np.zeros(27 * nd)
    for s, g in enumerate(gmap):
        if g >= 0:
            out[s * nd:(s + 1) * nd] = _np(t[g * nd:(g + 1) * nd])
    return out


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
