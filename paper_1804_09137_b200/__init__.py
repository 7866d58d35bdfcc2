"""B200-native TLR Gaussian log-likelihood (drop-in for tlrgeo's likelihood
and kriging path).  All numerics run in libtlrb200.so (sm_100a CUDA)."""
from .api import (  # noqa: F401
    DeviceError,
    Handle,
    LikelihoodConfig,
    LocationSet,
    MaternParams,
    NotPositiveDefiniteError,
    PredictionProblem,
    bessel_k,
    compress_tile,
    generate_locations,
    launch_count,
    log_likelihood,
    log_likelihood_parts,
    matern_block,
    predict,
    sample_measurements,
)

__all__ = [
    "DeviceError", "Handle", "LikelihoodConfig", "LocationSet", "MaternParams",
    "NotPositiveDefiniteError", "PredictionProblem", "bessel_k", "compress_tile",
    "generate_locations", "launch_count", "log_likelihood", "log_likelihood_parts",
    "matern_block", "predict", "sample_measurements",
]
