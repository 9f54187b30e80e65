"""B200-native (sm_100a) Ax / A^T b hot path of ctkrylov (arXiv 2211.14212).

The public names mirror the reference's C++ API (see api.py for the file:line map).
All compute runs in libctk_b200.so; importing this package does not touch the GPU.
"""
from .api import (  # noqa: F401
    BackprojectVariant,
    BeamMode,
    ConeGeometry,
    ConvergenceLog,
    CtkError,
    CudaError,
    DegenerateInputError,
    DimensionError,
    GeometryError,
    HybridStrategy,
    LambdaStrategy,
    NoiseModel,
    NumericalError,
    OperatorPair,
    ParameterError,
    PhantomKind,
    Projector,
    ProjectorKind,
    SolveResult,
    SolverOptions,
    StopReason,
    UnsupportedError,
    VolumeShape,
    ab_gmres,
    band_partition,
    ba_gmres,
    back_project,
    canonical_angle,
    cgls,
    cgls_tv,
    default_geometry,
    equidistant_angles,
    flsqr_tv,
    forward_project,
    hybrid_lsqr,
    launch_count,
    lsmr,
    lsqr,
    gradient,
    gradient_adjoint,
    tv_epsilon,
    tv_weights,
    augment_tikhonov,
    stack_weighted_gradient,
    make_phantom,
    add_noise,
    noise_rng_id,
    phantom_kind_from_string,
    projector_pair,
    shepp_logan_3d,
    sirt,
)
from ._lib import LIB_PATH, load  # noqa: F401


def bench_geometry(n: int, n_angles: int, nuv: int | None = None) -> ConeGeometry:
    """The BASELINE configs' acquisition: cone3d, h = 1, DSO = 2n,
    DOD = n, pixel 1.5, nu = nv = n, equidistant angles over [0, 2*pi)."""
    nuv = n if nuv is None else nuv
    return ConeGeometry(BeamMode.cone3d, 2.0 * n, 1.0 * n, 1.5, nuv, nuv, VolumeShape(n, n, n, 1.0),
                        equidistant_angles(n_angles))
