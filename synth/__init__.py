"""Seeded synthetic input generators shared by the oracle tests, the CUDA parity
tests and bench.py.

This package holds NO arithmetic of the method (no quartic, no ADMM update):
it only draws problem data (drive cycles, cost/loss coefficients, bounds,
demand scenarios, random quartics) in the boundary layout of include/admm.h.

Seeding contract: base seed 190310041; scenario j's
data depends only on (seed, j, n) -- never on q, the shard, or world size -- so
a rank that generates j in [j0, j1) gets exactly the rows the single-process
run would have.
"""

from .phev import (  # noqa: F401
    BASE_SEED,
    DELTA_E,
    E0_FRAC,
    E_MAX,
    EN_FRAC,
    battery_loss_coeffs,
    phev_problem,
    realised_drive,
    supervisor_problem,
    toy_problem,
    horizon_problem,
    random_problem,
)
from .quartics import quartic_family  # noqa: F401
