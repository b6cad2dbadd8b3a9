"""B200-native camera-covariance hot path of arXiv 1808.02414 (Polic,
Förstner, Pajdla): drop-in for the reference ``sfmcov::compute_covariance``.

The compute lives in ``libsfmcov_b200.so`` (hand-written sm_100a CUDA behind
the C ABI of include/sfmcov_b200.h); this package is the thin host mirror.
"""
from .sfmcov import (  # noqa: F401
    CovarianceDiagnostics,
    CovarianceOptions,
    CovarianceResult,
    Engine,
    Error,
    ErrorKind,
    FisherBlocks,
    ObservationIndex,
    Reconstruction,
    SparseJacobian,
    assemble_jacobian,
    build_fisher_blocks,
    build_observation_index,
    compute_covariance,
    default_engine,
    gauge_nullspace,
    schur_reduce,
    spd_inverse_blocks,
)
