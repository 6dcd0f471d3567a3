"""B200-native ADMM hot path of arXiv 1903.10041 (robust quadratic resource
allocation, exact quartic minimiser) -- fp64 sm_100a CUDA kernels behind a C
ABI (include/admm.h), driven from Python by argument marshalling only.

Importing this package loads libadmm_b200.so and fails loudly if it is
missing: there is no CPU path.
"""

from ._lib import (  # noqa: F401
    ADMM_BOX_EXACT,
    ADMM_BOX_PROJECT,
    ADMM_HIST_COLS,
    ADMM_NOT_CONVERGED,
    ADMM_OK,
    AdmmError,
    SO_PATH,
    admm_build_info,
    admm_create,
    admm_default_params,
    admm_destroy,
    admm_get_engine,
    admm_get_history,
    admm_get_params,
    admm_get_solution,
    admm_get_state,
    admm_get_timing,
    admm_iterate,
    admm_last_error,
    admm_nccl_unique_id,
    admm_reset,
    admm_set_params,
    admm_set_problem,
    admm_set_state,
    admm_solve,
    admm_workspace_bytes,
)
from .dist import dist_for, horizon_range, make_dist, shard_range  # noqa: F401
from .solver import AdmmSolver, quartic_minimize_batch  # noqa: F401
