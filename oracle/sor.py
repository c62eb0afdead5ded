"""Block SOR / SSOR in the red-black cell order (Alg. 3).

ORACLE (test infrastructure only). Two independent forms:

  `alg3`     Alg. 3 written out for a given traversal order rho = 1..m: the local defect uses the
             new values of the cells already visited and the old values of the others, with the
             diagonal block excluded (P:646 sums sigma != rho only), du = D^{-1} d is the new block
             value, u_rho <- (1 - omega) u_rho + omega du (LU solves).
  `sor_sweep` the coloured form the GPU runs: every red cell (colour (cx+cy+cz) mod 2 = 0) updated
             from the current u by u + omega D^{-1}(f - A u), then every black cell from the
             updated u; symmetric = forward (red, black) then backward (black, red) = SSOR
             (P:612-620).
Pinned equal to each other (reading #17) and to the invariants in tests/test_oracle_sor.py.
"""
from __future__ import annotations

import numpy as np

from .tier_b import TierB


def colour(tb: TierB, c: int) -> int:
    cx, cy, cz = tb.coords(c)
    return (cx + cy + cz) % 2


def red_black_order(tb: TierB, reverse: bool = False):
    N = tb.P.n_cells
    red = [c for c in range(N) if colour(tb, c) == 0]
    black = [c for c in range(N) if colour(tb, c) == 1]
    return black + red if reverse else red + black


def alg3(tb: TierB, u, f, omega, order):
    nd = tb.nd
    U = np.array(u, dtype=np.float64).reshape(-1, nd)
    F = np.asarray(f, dtype=np.float64).reshape(-1, nd)
    for c in order:
        d = F[c].copy()
        for nb, B in tb.nbr_blocks(c):          # sigma != rho: face neighbours only
            d -= B @ U[nb]
        du = np.linalg.solve(tb.diag_block(c), d)
        U[c] = (1.0 - omega) * U[c] + omega * du
    return U.reshape(-1)


def sor_sweep(tb: TierB, u, f, omega=1.0, symmetric=False):
    nd = tb.nd
    U = np.array(u, dtype=np.float64)
    seq = [0, 1, 1, 0] if symmetric else [0, 1]
    for col in seq:
        cells = [c for c in range(tb.P.n_cells) if colour(tb, c) == col]
        new = tb.sweep_cells(U, f, omega, cells)
        V = U.reshape(-1, nd)
        for r, c in enumerate(cells):
            V[c] = new[r]
    return U
