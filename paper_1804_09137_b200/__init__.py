"""B200-native TLR Gaussian log-likelihood (drop-in for tlrgeo's likelihood
and kriging path).  All numerics run in libtlrb200.so (sm_100a CUDA)."""
from .api import (  # noqa: F401
    EARTH_RADIUS_KM,
    DeviceError,
    Euclidean,
    GreatCircle,
    Handle,
    LikelihoodConfig,
    LocationSet,
    MaternParams,
    NotPositiveDefiniteError,
    PredictionProblem,
    bessel_k,
    close_handles,
    compress_tile,
    generate_locations,
    group_handle,
    launch_count,
    log_likelihood,
    log_likelihood_parts,
    matern_block,
    potrf_tile,
    predict,
    sample_measurements,
)
from .mle import EstimationError, EstimationResult, mle_fit  # noqa: F401
from .experiments import holdout_experiment, mc_experiment, mc_summaries, mse  # noqa: F401
from .dataio import (  # noqa: F401
    DataError,
    Dataset,
    load_dataset,
    partition_regions,
    save_dataset,
)

__all__ = [
    "EARTH_RADIUS_KM", "DeviceError", "Euclidean", "GreatCircle", "Handle", "LikelihoodConfig", "LocationSet", "MaternParams",
    "NotPositiveDefiniteError", "PredictionProblem", "bessel_k", "close_handles", "compress_tile",
    "generate_locations", "group_handle", "launch_count", "log_likelihood", "log_likelihood_parts",
    "matern_block", "potrf_tile", "predict", "sample_measurements",
    "DataError", "Dataset", "load_dataset", "partition_regions", "save_dataset",
    "EstimationError", "EstimationResult", "mle_fit",
    "holdout_experiment", "mc_experiment", "mc_summaries", "mse",
]
