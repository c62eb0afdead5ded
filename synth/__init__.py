"""Seeded synthetic inputs shared by the oracle and the product path (no DG arithmetic)."""
from .problem import (DIRICHLET, NEUMANN, Problem, make_config, make_vectors,
                      random_problem, config_seed, CONFIG_INDEX)
from .rng import normal, splitmix64, uniform_pm1

__all__ = ["DIRICHLET", "NEUMANN", "Problem", "make_config", "make_vectors", "random_problem",
           "config_seed", "CONFIG_INDEX", "normal", "splitmix64", "uniform_pm1"]
