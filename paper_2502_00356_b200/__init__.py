"""B200-native (sm_100a) BesselK evaluation and Matern covariance generation.

Drop-in for the reference package ``besselgp`` (arXiv 2502.00356): the names of
/root/reference/pkg/src/besselgp/__init__.py:3-33 with the same semantics,
plus the SPEC's covariance-engine API and GPU batch entry points.  All numeric
work runs in libbesselgp_sm100a.so (CUDA, sm_100a); there is no CPU fallback.
"""

from .besselk import (
    DEFAULT_CONFIG,
    EPS_MACHINE,
    VALIDATED_NU_MAX,
    VALIDATED_X_MAX,
    BatchResult,
    BesselResult,
    DomainError,
    EvalPoint,
    PathTaken,
    QuadratureConfig,
    bessel_k,
    bessel_k_batch,
    bessel_k_integral,
    bessel_k_series,
    fixed_window_log_bessel_k,
    log_integrand,
    log_integrand_d1,
    log_integrand_d2,
    temme_pair,
    temme_sums_batch,
)
from .covariance import (
    CovarianceMatrix,
    LocationSet,
    MaternParams,
    Ordering,
    TileSpec,
    empty_host_matrix,
    generate_covariance,
    generate_tile,
    lower_tile_count,
    matern,
    matern_batch,
    matern_plan,
    matern_tile,
    morton_order,
    normalize_locations,
)
from ._lib import BackendError, BackendUnavailable
from . import distributed, gp

__all__ = [
    # reference besselgp/__init__.py:19-33
    "BesselResult",
    "DomainError",
    "EvalPoint",
    "PathTaken",
    "QuadratureConfig",
    "bessel_k",
    "bessel_k_integral",
    "bessel_k_series",
    "fixed_window_log_bessel_k",
    "log_integrand",
    "log_integrand_d1",
    "log_integrand_d2",
    "temme_pair",
    # SPEC covariance engine
    "CovarianceMatrix",
    "LocationSet",
    "MaternParams",
    "Ordering",
    "TileSpec",
    "generate_covariance",
    "generate_tile",
    "matern",
    "matern_tile",
    "morton_order",
    "normalize_locations",
    # GPU batch / plumbing
    "BatchResult",
    "BackendError",
    "BackendUnavailable",
    "DEFAULT_CONFIG",
    "EPS_MACHINE",
    "VALIDATED_NU_MAX",
    "VALIDATED_X_MAX",
    "bessel_k_batch",
    "empty_host_matrix",
    "lower_tile_count",
    "matern_batch",
    "matern_plan",
    "temme_sums_batch",
]

__version__ = "0.1.0"
