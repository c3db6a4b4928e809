"""B200-native (sm_100a) exact-likelihood engine behind Fisher-BT (arXiv 2601.11437).

Drop-in for the hot path of the reference package ``maternmle``
(``pkg/src/maternmle/__init__.py:7-110``): the same names and signatures for the
covariance, log-likelihood, score/Fisher and Fisher-BT entry points, computed by
hand-written CUDA kernels behind the C ABI in ``include/maternfisher.h``.
Importing the package loads ``libmaternfisher.so``; there is no CPU fallback.
"""

from .batch import BatchCoordinator, BatchedObjective, eval_batch, fit_many
from .bessel import (
    BesselRegime,
    MidRangeSmallOrderWarning,
    bessel_k,
    case2_series,
    case3_series,
    case4_series,
    digamma,
    dnu_xnu_knu,
    select_regime,
    u_poly_coeffs,
)
from .datasets import WORKLOADS, Workload, gmm_locations, jittered_grid, simulate_field
from .engine import Engine
from .fisher_bt import (
    FisherBTConfig,
    InitializationFailed,
    LikelihoodObjective,
    OptResult,
    SingularInformation,
    Termination,
    armijo_relaxed,
    fisher_bt,
    fisher_step,
    l9_candidates,
    nelder_mead,
    objective_for,
    select_initial,
)
from .likelihood import (
    LikelihoodEval,
    NotPositiveDefinite,
    cholesky_lower,
    grad_and_fisher,
    log_likelihood,
    trace_product,
)
from .matern import (
    MaternParams,
    SpatialDataset,
    build_cov_matrix,
    build_dcov_matrix,
    dcov_dalpha,
    dcov_dnu,
    dcov_dsigma2,
    matern_cov,
)
from .simulate import (
    GENERATOR_ID,
    LocationScheme,
    PlanError,
    SimulationPlan,
    gen_locations,
    microergodic,
    replicate_seed,
    simulate_grf,
)
from ._native import device_count, release_cached_memory, LIB_PATH

__version__ = "0.1.0"

__all__ = [
    "BatchCoordinator", "BatchedObjective", "eval_batch", "fit_many",
    "BesselRegime", "MidRangeSmallOrderWarning", "bessel_k", "case2_series", "case3_series",
    "case4_series", "digamma", "dnu_xnu_knu", "select_regime", "u_poly_coeffs",
    "GENERATOR_ID", "LocationScheme", "PlanError", "SimulationPlan", "gen_locations",
    "microergodic", "replicate_seed", "simulate_grf",
    "WORKLOADS", "Workload", "gmm_locations", "jittered_grid", "simulate_field",
    "Engine",
    "FisherBTConfig", "InitializationFailed", "LikelihoodObjective", "OptResult",
    "SingularInformation", "Termination", "armijo_relaxed", "fisher_bt", "fisher_step",
    "l9_candidates", "nelder_mead", "objective_for", "select_initial",
    "LikelihoodEval", "NotPositiveDefinite", "cholesky_lower", "grad_and_fisher",
    "log_likelihood", "trace_product",
    "MaternParams", "SpatialDataset", "build_cov_matrix", "build_dcov_matrix",
    "dcov_dalpha", "dcov_dnu", "dcov_dsigma2", "matern_cov",
    "device_count", "release_cached_memory", "LIB_PATH", "__version__",
]
