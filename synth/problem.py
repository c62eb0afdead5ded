"""Problem description + the BASELINE.json configs C1..C5 as seeded synthetic inputs.

Pure data: mesh sizes, degree, penalty parameter, per-cell coefficients,
boundary-condition flags and the seeded u / f vectors. No DG arithmetic lives
here (that is in `oracle/` and in the CUDA library, independently).

Recipes (SURVEY.md §8(c) readings #1, #10, #11, #19, #20 and §8(d)):
  seed_k = 180511930 + k;  u = SplitMix64(seed_k);  f = SplitMix64(seed_k ^ GOLDEN);
  coefficients = SplitMix64(seed_k + 2).  u, f i.i.d. U[-1, 1).
  C1  8^3 on [0,1]^3,  p=2, K=1, alpha=2, all Dirichlet        (BASELINE configs[0])
  C2 32^3 on [0,1]^3,  p=3, K=1, alpha=2, all Dirichlet        (BASELINE configs[1])
  C3 64^3 on [0,1]^3,  p=4, K_T = exp(g_T), g ~ N(0, 2^2)      (BASELINE configs[2])
  C4 64^3 on [0,1]^3,  p=3, K=1e-3, b=(1,.5,.25), BiCGStab     (BASELINE configs[3])
  C5 60x220x85 on 1200x2200x170, p=2, K=diag(kx,kx,0.1kx),
     log10 kx = clip(1.5*(sqrt(.5) L_k + sqrt(.5) xi), -3, 4.3),
     Neumann on z=0 / z=Lz, Dirichlet elsewhere                 (BASELINE configs[4])
C5 is a synthetic stand-in for the SPE10 permeability field (the dataset is not
in this container); no dataset value is reproduced.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .rng import GOLDEN, normal, uniform_pm1

DIRICHLET = 0
NEUMANN = 1

BASE_SEED = 180511930


@dataclasses.dataclass
class Problem:
    nx: int
    ny: int
    nz: int
    p: int
    Lx: float = 1.0
    Ly: float = 1.0
    Lz: float = 1.0
    alpha: float = 2.0
    # per-cell diffusion: shape (N,) scalar or (N, 3) diagonal; cell c = cx + nx*(cy + ny*cz)
    K: np.ndarray = None
    b: tuple = (0.0, 0.0, 0.0)          # constant advection
    b_cells: Optional[np.ndarray] = None  # per-cell advection (N, 3); overrides b when set
    c: Optional[np.ndarray] = None      # per-cell reaction (N,) or None
    bc: tuple = (DIRICHLET,) * 6        # x-, x+, y-, y+, z-, z+
    name: str = "custom"
    local_solver: str = "cg"            # "cg" (b = 0) or "bicgstab"

    @property
    def n(self) -> int:
        return self.p + 1

    @property
    def nd(self) -> int:
        return self.n ** 3

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_dof(self) -> int:
        return self.n_cells * self.nd

    @property
    def h(self) -> tuple:
        return (self.Lx / self.nx, self.Ly / self.ny, self.Lz / self.nz)

    def K3(self) -> np.ndarray:
        """Per-cell diagonal of K as (N, 3)."""
        K = np.asarray(self.K, dtype=np.float64)
        if K.ndim == 1:
            return np.repeat(K[:, None], 3, axis=1)
        return K

    def b3(self) -> np.ndarray:
        """Per-cell advection as (N, 3): b_cells, else the constant b on every cell."""
        if self.b_cells is not None:
            return np.asarray(self.b_cells, dtype=np.float64).reshape(self.n_cells, 3)
        return np.tile(np.asarray(self.b, dtype=np.float64), (self.n_cells, 1))

    def has_convection(self) -> bool:
        return bool(np.any(self.b3() != 0.0))

    def c_cells(self) -> np.ndarray:
        if self.c is None:
            return np.zeros(self.n_cells)
        return np.asarray(self.c, dtype=np.float64)


def config_seed(k: int) -> int:
    return BASE_SEED + k


def u_stream(seed: int) -> int:
    return seed


def f_stream(seed: int) -> int:
    return seed ^ int(GOLDEN)


def coef_stream(seed: int) -> int:
    return seed + 2


def make_config(name: str) -> Problem:
    """The BASELINE.json configs as Problems (coefficients generated, vectors not)."""
    name = name.upper()
    if name == "C1":
        P = Problem(8, 8, 8, 2, alpha=2.0, name="C1")
        P.K = np.ones(P.n_cells)
    elif name == "C2":
        P = Problem(32, 32, 32, 3, alpha=2.0, name="C2")
        P.K = np.ones(P.n_cells)
    elif name == "C3":
        P = Problem(64, 64, 64, 4, alpha=2.0, name="C3")
        g = 2.0 * normal(coef_stream(config_seed(3)), 0, P.n_cells)
        P.K = np.exp(g)
    elif name == "C4":
        P = Problem(64, 64, 64, 3, alpha=2.0, name="C4", b=(1.0, 0.5, 0.25),
                    local_solver="bicgstab")
        P.K = np.full(P.n_cells, 1e-3)
    elif name == "C5":
        P = Problem(60, 220, 85, 2, Lx=1200.0, Ly=2200.0, Lz=170.0, alpha=2.0, name="C5",
                    bc=(DIRICHLET, DIRICHLET, DIRICHLET, DIRICHLET, NEUMANN, NEUMANN))
        s = coef_stream(config_seed(5))
        layer = normal(s, 0, P.nz)                       # L_k, one per z-layer
        xi = normal(s, P.nz, P.n_cells)                  # i.i.d. per cell
        cz = np.arange(P.n_cells) // (P.nx * P.ny)
        lg = np.clip(1.5 * (np.sqrt(0.5) * layer[cz] + np.sqrt(0.5) * xi), -3.0, 4.3)
        kx = 10.0 ** lg
        P.K = np.stack([kx, kx, 0.1 * kx], axis=1)
    else:
        raise ValueError(f"unknown config {name}")
    return P


CONFIG_INDEX = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}


def make_vectors(P: Problem, seed: Optional[int] = None, cell_begin: int = 0,
                 cell_end: Optional[int] = None):
    """Seeded u, f (U[-1,1)) for cells [cell_begin, cell_end), in the global DoF order."""
    if seed is None:
        seed = config_seed(CONFIG_INDEX.get(P.name, 0))
    if cell_end is None:
        cell_end = P.n_cells
    start = cell_begin * P.nd
    count = (cell_end - cell_begin) * P.nd
    return uniform_pm1(u_stream(seed), start, count), uniform_pm1(f_stream(seed), start, count)


def random_problem(nx, ny, nz, p, seed, *, aniso=True, b=(0.0, 0.0, 0.0), c=False,
                   bc=(DIRICHLET,) * 6, alpha=2.0, L=(1.0, 1.0, 1.0), spread=1.0):
    """Small random test problem: K = exp(spread * N(0,1)) per cell and component."""
    P = Problem(nx, ny, nz, p, Lx=L[0], Ly=L[1], Lz=L[2], alpha=alpha, b=tuple(b), bc=tuple(bc))
    N = P.n_cells
    g = normal(seed, 0, 3 * N).reshape(N, 3)
    if aniso:
        P.K = np.exp(spread * g)
    else:
        P.K = np.exp(spread * g[:, 0])
    if c:
        P.c = np.exp(normal(seed + 7, 0, N))
    P.local_solver = "cg" if tuple(b) == (0.0, 0.0, 0.0) else "bicgstab"
    return P
