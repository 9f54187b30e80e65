"""Python mirror of the reference's public API for the Ax / A^T b hot path.

Names, argument meaning and error behaviour follow ctkrylov (/root/reference/proj):

=====================================  ==================================================
this module                            reference
=====================================  ==================================================
``BeamMode``, ``ConeGeometry``         geometry.hpp:11, 24-55
``equidistant_angles``                 geometry.hpp:57-64
``default_geometry``                   geometry.hpp:66-87
``canonical_angle``                    types.hpp:172-177
``VolumeShape``                        types.hpp:35-41
error classes                          types.hpp:14-31
``BackprojectVariant``                 projector.hpp:16
``forward_project`` / ``back_project`` projector.hpp:134-162, 283-297
``OperatorPair`` / ``projector_pair``  operators.hpp:18-45, 91-115
``SolverOptions`` / ``SolveResult``    solve_log.hpp:28-76
``cgls`` ``lsqr`` ``lsmr``             solvers.hpp:13-231
``HybridStrategy`` / ``hybrid_lsqr``   hybrid.hpp:15-33, 76-116
``cgls_tv``                            tv.hpp:45-110
``PhantomKind`` / ``make_phantom``     phantom.hpp:13, 118-152
``NoiseModel`` / ``add_noise``         noise.hpp:10-47
``gradient`` / ``gradient_adjoint``    gradient.hpp:9-54
``tv_epsilon`` / ``tv_weights``        tv.hpp:17-43
``augment_tikhonov``                   operators.hpp:118-139
``stack_weighted_gradient``            operators.hpp:141-186
=====================================  ==================================================

Every computation runs in libctk_b200.so (sm_100a kernels + C++ solvers) through the
C-ABI; there is no CPU path.  Host (numpy) inputs use the OperatorPair host-span
semantics (copies in and out per call); CUDA torch tensors use the device-resident entry
points.  dtype float32 selects the performance kernels, float64 the exact-parity kernels.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L


# ---- errors (types.hpp:14-31) --------------------------------------------------------------
class CtkError(RuntimeError):
    pass


class DimensionError(CtkError):
    pass


class GeometryError(CtkError):
    pass


class ParameterError(CtkError):
    pass


class DegenerateInputError(CtkError):
    pass


class NumericalError(CtkError):
    def __init__(self, msg, iteration):
        super().__init__(msg)
        self.iteration = iteration


class CudaError(CtkError):
    pass


class UnsupportedError(CtkError):
    pass


_ERR = {
    L.CTK_E_DIMENSION: DimensionError,
    L.CTK_E_GEOMETRY: GeometryError,
    L.CTK_E_PARAMETER: ParameterError,
    L.CTK_E_DEGENERATE: DegenerateInputError,
    L.CTK_E_CUDA: CudaError,
    L.CTK_E_UNSUPPORTED: UnsupportedError,
}


def _check(rc):
    if rc == L.CTK_OK:
        return
    code, msg, it = L.last_error()
    if rc == L.CTK_E_NUMERICAL:
        raise NumericalError(msg, it)
    raise _ERR.get(rc, CtkError)(msg)


# ---- geometry -------------------------------------------------------------------------------
class BeamMode(IntEnum):
    parallel2d = 0
    parallel3d = 1
    cone3d = 2


class BackprojectVariant(IntEnum):
    matched = 0
    voxel_driven = 1


class ProjectorKind(IntEnum):
    joseph = 0
    siddon = 1


class PhantomKind(IntEnum):
    """phantom.hpp:13."""
    shepp_logan_3d = 0
    shepp_logan_2d = 1
    piecewise_blocks = 2


def phantom_kind_from_string(s: str) -> PhantomKind:
    """phantom.hpp:147-152."""
    try:
        return PhantomKind[s]
    except KeyError:
        raise ParameterError("unknown phantom kind: " + s) from None


class StopReason(IntEnum):
    max_iters = 0
    residual_increase = 1
    tolerance = 2
    breakdown = 3


class LambdaStrategy(IntEnum):
    fixed = 0
    dp = 1
    gcv = 2


TWO_PI = 2.0 * math.pi


def canonical_angle(a: float) -> float:
    r = math.fmod(a, TWO_PI)
    if r < 0.0:
        r += TWO_PI
    return r


@dataclass
class VolumeShape:
    nx: int = 0
    ny: int = 0
    nz: int = 0
    spacing: float = 1.0

    def size(self) -> int:
        return self.nx * self.ny * self.nz


@dataclass
class ConeGeometry:
    mode: BeamMode = BeamMode.parallel2d
    source_to_origin: float = 0.0
    origin_to_detector: float = 0.0
    detector_pixel_size: float = 1.0
    nu: int = 0
    nv: int = 0
    vol: VolumeShape = field(default_factory=VolumeShape)
    angles: Sequence[float] = field(default_factory=list)

    def proj_shape(self):
        return (len(self.angles), self.nu, self.nv)

    def validate(self):
        """ConeGeometry::validate (geometry.hpp:35-54)."""
        v = self.vol
        if len(self.angles) == 0:
            raise GeometryError("geometry needs at least one angle")
        if self.nu <= 0 or self.nv <= 0:
            raise GeometryError("detector pixel counts must be positive")
        if not self.detector_pixel_size > 0.0:
            raise GeometryError("detector pixel size must be positive")
        if not self.origin_to_detector > 0.0:
            raise GeometryError("origin-to-detector distance must be positive")
        if v.nx <= 0 or v.ny <= 0 or v.nz <= 0 or not v.spacing > 0.0:
            raise GeometryError("geometry volume descriptor invalid")
        if self.mode == BeamMode.parallel2d and (v.nz != 1 or self.nv != 1):
            raise GeometryError("parallel2d requires nz = 1 and nv = 1")
        if self.mode == BeamMode.cone3d:
            if not self.source_to_origin > 0.0:
                raise GeometryError("cone3d requires a positive source-to-origin distance")
            hx, hy, hz = 0.5 * v.nx * v.spacing, 0.5 * v.ny * v.spacing, 0.5 * v.nz * v.spacing
            if self.source_to_origin <= math.sqrt(hx * hx + hy * hy + hz * hz):
                raise GeometryError("cone3d source lies inside the volume diagonal")

    def desc(self):
        ang = np.ascontiguousarray(np.asarray(self.angles, dtype=np.float64))
        d = L.GeomDesc(int(self.mode), float(self.source_to_origin), float(self.origin_to_detector),
                       float(self.detector_pixel_size), int(self.nu), int(self.nv), int(self.vol.nx),
                       int(self.vol.ny), int(self.vol.nz), float(self.vol.spacing), len(ang),
                       ang.ctypes.data_as(C.POINTER(C.c_double)))
        d._keep = ang
        return d

    def subset(self, first: int, count: int) -> "ConeGeometry":
        return ConeGeometry(self.mode, self.source_to_origin, self.origin_to_detector, self.detector_pixel_size,
                            self.nu, self.nv, VolumeShape(self.vol.nx, self.vol.ny, self.vol.nz, self.vol.spacing),
                            list(np.asarray(self.angles, dtype=np.float64)[first:first + count]))


def band_partition(geom: ConeGeometry, z0s, nzs):
    """The band-sharded range's row partition (ctk_band_partition): per slab, the detector
    rows its rays reach [t0, t1) and the rows its rank owns [o0, o1)."""
    lib = L.load()
    R = len(z0s)
    arr = lambda v: (C.c_int * R)(*v)
    t0, t1, o0, o1 = arr([0] * R), arr([0] * R), arr([0] * R), arr([0] * R)
    _check(lib.ctk_band_partition(C.byref(geom.desc()), R, arr(z0s), arr(nzs), t0, t1, o0, o1))
    return [list(x) for x in (t0, t1, o0, o1)]


def equidistant_angles(n: int, start_rad: float = 0.0, range_rad: float = TWO_PI):
    """geometry.hpp:57-64."""
    if n <= 0:
        raise GeometryError("angle count must be positive")
    return [canonical_angle(start_rad + range_rad * i / n) for i in range(n)]


def default_geometry(mode: BeamMode, vol: VolumeShape, n_angles: int, range_rad: float = TWO_PI) -> ConeGeometry:
    """geometry.hpp:66-87."""
    g = ConeGeometry(mode=BeamMode(mode), vol=vol, angles=equidistant_angles(n_angles, 0.0, range_rad))
    n = max(vol.nx, vol.ny, vol.nz)
    if g.mode == BeamMode.cone3d:
        g.source_to_origin = 2.0 * n * vol.spacing
        g.origin_to_detector = 1.0 * n * vol.spacing
        g.detector_pixel_size = 1.5 * vol.spacing
        g.nu = g.nv = (3 * n) // 2
    else:
        g.origin_to_detector = 1.0 * n * vol.spacing
        g.detector_pixel_size = vol.spacing
        g.nu = (3 * n) // 2
        g.nv = 1 if g.mode == BeamMode.parallel2d else (3 * vol.nz) // 2
    g.validate()
    return g


# ---- native projector handle ----------------------------------------------------------------
def _is_torch_cuda(a) -> bool:
    return type(a).__module__.startswith("torch") and getattr(a, "is_cuda", False)


def _numel(a) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _torch_stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Projector:
    """Owns one native ctk_geom handle (validated geometry + device tables + workspace)."""

    def __init__(self, geom: ConeGeometry, projector: ProjectorKind = ProjectorKind.joseph, bp_partitions: int = 1):
        geom.validate()
        self.geom = geom
        self.lib = L.load()
        h = C.c_void_p()
        _check(self.lib.ctk_geom_create(C.byref(geom.desc()), C.byref(h)))
        self.handle = h
        if projector != ProjectorKind.joseph:
            _check(self.lib.ctk_geom_set_projector(h, int(projector)))
        if bp_partitions != 1:
            _check(self.lib.ctk_geom_set_bp_partitions(h, int(bp_partitions)))
        ds, rs = C.c_size_t(), C.c_size_t()
        _check(self.lib.ctk_geom_sizes(h, C.byref(ds), C.byref(rs)))
        self.domain_size, self.range_size = ds.value, rs.value
        self._comm = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.ctk_geom_destroy(h)
            self.handle = None

    def set_slab(self, z0: int, nz_local: int):
        """Domain vectors hold slices [z0, z0 + nz_local) of the volume (z-slab sharding);
        nz_local = 0 restores the whole volume."""
        _check(self.lib.ctk_geom_set_slab(self.handle, int(z0), int(nz_local)))
        ds, rs = C.c_size_t(), C.c_size_t()
        _check(self.lib.ctk_geom_sizes(self.handle, C.byref(ds), C.byref(rs)))
        self.domain_size, self.range_size = ds.value, rs.value

    def attach_comm(self, comm):
        _check(self.lib.ctk_geom_attach_comm(self.handle, comm.handle))
        self._comm = comm

    def shard_range(self):
        """Band-sharded range (z-slab + communicator, collective): range vectors hold this
        rank's detector-row window (range_rows) with the rows it does not own at zero."""
        _check(self.lib.ctk_geom_shard_range(self.handle))
        ds, rs = C.c_size_t(), C.c_size_t()
        _check(self.lib.ctk_geom_sizes(self.handle, C.byref(ds), C.byref(rs)))
        self.domain_size, self.range_size = ds.value, rs.value

    def range_rows(self):
        """(w0, nw, o0, no): rows held [w0, w0 + nw) and owned [o0, o0 + no)."""
        v = [C.c_int() for _ in range(4)]
        _check(self.lib.ctk_geom_range_rows(self.handle, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def local_range(self, y_full):
        """The held rows of a whole-range vector [n_angles][nv][nu], non-owned rows zeroed
        (the layout of this rank's range vectors under the band-sharded range)."""
        w0, nw, o0, no = self.range_rows()
        g = self.geom
        yv = y_full.reshape(len(g.angles), g.nv, g.nu)
        out = yv[:, w0:w0 + nw, :].copy() if isinstance(yv, np.ndarray) else yv[:, w0:w0 + nw, :].clone()
        out[:, :o0 - w0, :] = 0
        out[:, o0 - w0 + no:, :] = 0
        return out.reshape(-1)

    def last_kernel_ms(self) -> float:
        return float(self.lib.ctk_geom_last_kernel_ms(self.handle))

    @staticmethod
    def _suffix(dtype):
        dt = np.dtype(str(dtype).replace("torch.", ""))
        if dt == np.float32:
            return "f32"
        if dt == np.float64:
            return "f64"
        raise ParameterError(f"unsupported dtype {dtype}; use float32 or float64")

    @staticmethod
    def _check_buffers(a, b):
        """Both operands CUDA tensors or both host arrays, one dtype, contiguous: the native
        entry points read and write them as flat arrays."""
        dev = _is_torch_cuda(a)
        if dev != _is_torch_cuda(b):
            raise ParameterError("input and output must both be CUDA tensors or both host arrays")
        if a.dtype != b.dtype:
            raise ParameterError(f"input and output dtypes differ ({a.dtype} vs {b.dtype})")
        for v in (a, b):
            if not (v.is_contiguous() if dev else (isinstance(v, np.ndarray) and v.flags.c_contiguous
                                                   and v.dtype.isnative)):
                raise ParameterError("operator buffers must be contiguous (native byte order)")

    def forward(self, x, y, stream=None):
        """y <- A x (overwrites y).  numpy -> host entry point; CUDA tensors -> device."""
        if _numel(x) != self.domain_size or _numel(y) != self.range_size:
            raise DimensionError("operator domain size mismatch")
        self._check_buffers(x, y)
        t = self._suffix(x.dtype)
        if _is_torch_cuda(x):
            _check(getattr(self.lib, f"ctk_ax_{t}")(self.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                                     stream if stream is not None else _torch_stream()))
        else:
            _check(getattr(self.lib, f"ctk_ax_host_{t}")(self.handle, x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p)))

    def back(self, y, x, variant=BackprojectVariant.matched, stream=None):
        if _numel(y) != self.range_size or _numel(x) != self.domain_size:
            raise DimensionError("operator range size mismatch")
        self._check_buffers(y, x)
        t = self._suffix(y.dtype)
        if _is_torch_cuda(y):
            _check(getattr(self.lib, f"ctk_atb_{t}")(self.handle, int(variant), C.c_void_p(y.data_ptr()),
                                                      C.c_void_p(x.data_ptr()), stream if stream is not None else _torch_stream()))
        else:
            _check(getattr(self.lib, f"ctk_atb_host_{t}")(self.handle, int(variant), y.ctypes.data_as(C.c_void_p),
                                                           x.ctypes.data_as(C.c_void_p)))

    def forward_pair(self, x1, y1, x2, y2, stream=None):
        """y1 <- A x1 and y2 <- A x2 in one ray march (float32 CUDA tensors, Joseph or Siddon,
        whole-volume handle); each output bit-identical to forward()."""
        for x, y in ((x1, y1), (x2, y2)):
            if _numel(x) != self.domain_size or _numel(y) != self.range_size:
                raise DimensionError("operator domain size mismatch")
            if not _is_torch_cuda(x):
                raise ParameterError("forward_pair takes CUDA tensors")
            self._check_buffers(x, y)
            if str(x.dtype) != "torch.float32":
                raise ParameterError("forward_pair is float32")
        _check(self.lib.ctk_ax_pair_f32(self.handle, C.c_void_p(x1.data_ptr()), C.c_void_p(y1.data_ptr()),
                                        C.c_void_p(x2.data_ptr()), C.c_void_p(y2.data_ptr()),
                                        stream if stream is not None else _torch_stream()))

    def residual2(self, x, b) -> float:
        """||A x - b||^2 without storing A x (float32 CUDA tensors)."""
        out = C.c_double()
        _check(self.lib.ctk_ax_residual_f32(self.handle, C.c_void_p(x.data_ptr()), C.c_void_p(b.data_ptr()),
                                            C.byref(out), _torch_stream()))
        return out.value


def _empty_like(a, n):
    if _is_torch_cuda(a):
        import torch

        return torch.empty(n, dtype=a.dtype, device=a.device)
    return np.empty(n, dtype=a.dtype)


def _contiguous(a):
    """apply_forward/apply_back take any array-like (the reference's spans are contiguous):
    CUDA tensors are made contiguous on the device, everything else becomes a contiguous
    host array in native byte order."""
    if _is_torch_cuda(a):
        return a if a.is_contiguous() else a.contiguous()
    a = np.asarray(a)
    if not a.dtype.isnative:
        a = a.astype(a.dtype.newbyteorder("="))
    return np.ascontiguousarray(a)


def _host(a, dtype=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


# ---- OperatorPair (operators.hpp:18-45) -----------------------------------------------------
@dataclass
class OperatorPair:
    domain_size: int
    range_size: int
    matched: bool
    domain_shape: VolumeShape
    forward: Callable  # forward(x, y): y <- A x, overwrites y
    back: Callable     # back(y, x):   x <- B y, overwrites x
    dtype: np.dtype = np.dtype(np.float32)
    projector: Optional[Projector] = None
    variant: BackprojectVariant = BackprojectVariant.matched

    def check_domain(self, n):
        if n != self.domain_size:
            raise DimensionError("operator domain size mismatch")

    def check_range(self, n):
        if n != self.range_size:
            raise DimensionError("operator range size mismatch")

    def apply_forward(self, x):
        x = _contiguous(x)
        self.check_domain(x.size if isinstance(x, np.ndarray) else x.numel())
        y = _empty_like(x, self.range_size)
        self.forward(x, y)
        return y

    def apply_back(self, y):
        y = _contiguous(y)
        self.check_range(y.size if isinstance(y, np.ndarray) else y.numel())
        x = _empty_like(y, self.domain_size)
        self.back(y, x)
        return x


def projector_pair(geom: ConeGeometry, variant: BackprojectVariant = BackprojectVariant.matched,
                   dtype=np.float32, projector: ProjectorKind = ProjectorKind.joseph,
                   bp_partitions: int = 1, slab: Optional[Tuple[int, int]] = None, comm=None,
                   shard_range: bool = False) -> OperatorPair:
    """operators.hpp:91-115 -- the projector pair of a geometry, backed by the sm_100a kernels.
    slab = (z0, nz_local): the pair acts on slices [z0, z0 + nz_local) of the volume
    (z-slab sharding; f32 Joseph operators).  comm: attach a communicator; shard_range (with
    a slab): the band-sharded range -- range vectors hold this rank's detector-row window
    (Projector.range_rows / local_range)."""
    geom.validate()
    canon = ConeGeometry(geom.mode, geom.source_to_origin, geom.origin_to_detector, geom.detector_pixel_size,
                         geom.nu, geom.nv, geom.vol, [canonical_angle(a) for a in geom.angles])
    proj = Projector(canon, projector, bp_partitions)
    shape = canon.vol
    if slab is not None:
        proj.set_slab(*slab)
        shape = VolumeShape(canon.vol.nx, canon.vol.ny, int(slab[1]), canon.vol.spacing)
    if comm is not None:
        proj.attach_comm(comm)
        if shard_range:
            proj.shard_range()
    v = BackprojectVariant(variant)
    return OperatorPair(proj.domain_size, proj.range_size, v == BackprojectVariant.matched, shape,
                        lambda x, y: proj.forward(x, y), lambda y, x: proj.back(y, x, v), np.dtype(dtype), proj, v)


def forward_project(vol, geom: ConeGeometry):
    """projector.hpp:134-162.  Returns the projections as [n_angles, nv, nu]."""
    p = Projector(geom)
    x = vol if _is_torch_cuda(vol) else _host(vol).reshape(-1)
    if _is_torch_cuda(x):
        x = x.reshape(-1)
    y = _empty_like(x, p.range_size)
    p.forward(x, y)
    return y.reshape(len(geom.angles), geom.nv, geom.nu)


def back_project(proj, geom: ConeGeometry, variant: BackprojectVariant = BackprojectVariant.matched):
    """projector.hpp:283-297.  Returns the volume as [nz, ny, nx]."""
    n = (proj.size if isinstance(proj, np.ndarray) else proj.numel())
    if n != len(geom.angles) * geom.nu * geom.nv:
        raise DimensionError("projection shape does not match geometry descriptor")
    p = Projector(geom)
    y = proj.reshape(-1) if _is_torch_cuda(proj) else _host(proj).reshape(-1)
    x = _empty_like(y, p.domain_size)
    p.back(y, x, variant)
    return x.reshape(geom.vol.nz, geom.vol.ny, geom.vol.nx)


# ---- solvers --------------------------------------------------------------------------------
@dataclass
class SolverOptions:
    max_iters: int = 100
    stop_on_explicit_residual_increase: bool = True
    residual_tolerance: float = 1e-6
    reorth: bool = True
    ground_truth: Optional[np.ndarray] = None
    rng_seed: int = 0
    iterate_observer: Optional[Callable[[int, np.ndarray], None]] = None

    def validate(self):
        if self.max_iters < 1:
            raise ParameterError("max_iters must be >= 1")
        if self.residual_tolerance < 0.0:
            raise ParameterError("residual tolerance must be >= 0")


@dataclass
class ConvergenceLog:
    implicit_residual: list
    explicit_residual: list
    relative_error: list
    lambda_: list
    solver: str
    precision: str
    matched: bool

    def iterations(self):
        return len(self.explicit_residual)


@dataclass
class SolveResult:
    x: object
    shape: VolumeShape
    iterations_run: int
    stop_reason: StopReason
    log: ConvergenceLog
    outer_starts: list = field(default_factory=list)
    stored_domain_basis: int = 0
    stored_range_basis: int = 0
    warnings: list = field(default_factory=list)


@dataclass
class HybridStrategy:
    kind: LambdaStrategy = LambdaStrategy.fixed
    lambda_: float = 0.0
    noise_level: float = 0.0

    @staticmethod
    def fixed(lam: float) -> "HybridStrategy":
        if lam < 0.0:
            raise ParameterError("fixed lambda must be nonnegative")
        return HybridStrategy(LambdaStrategy.fixed, lam, 0.0)

    @staticmethod
    def dp(noise_level: float) -> "HybridStrategy":
        if not (0.0 < noise_level < 1.0):
            raise ParameterError("dp strategy needs a noise level in (0,1)")
        return HybridStrategy(LambdaStrategy.dp, 0.0, noise_level)

    @staticmethod
    def gcv() -> "HybridStrategy":
        return HybridStrategy(LambdaStrategy.gcv, 0.0, 0.0)


_SOLVER_ID = {"cgls": 0, "lsqr": 1, "lsmr": 2, "hybrid_lsqr": 3, "cgls_tv": 4, "sirt": 5, "ab_gmres": 6,
              "ba_gmres": 7, "flsqr_tv": 8}


def _solve(name, pair: OperatorPair, b, opts: SolverOptions, lam=0.0, strategy=None, outer=1, inner=1, warm=False):
    opts.validate()
    if pair.projector is None:
        raise ParameterError(f"{name}: the device solvers need a projector_pair (sm_100a operators)")
    n_b = b.size if isinstance(b, np.ndarray) else b.numel()
    pair.check_range(n_b)
    proj = pair.projector
    lib = proj.lib
    dev = _is_torch_cuda(b)
    if dev and not b.is_contiguous():
        b = b.contiguous()
    t = Projector._suffix(b.dtype)
    ndt = np.float32 if t == "f32" else np.float64
    cap = outer * inner if name == "cgls_tv" else opts.max_iters
    bufs = [np.zeros(cap + 1) for _ in range(4)]
    starts = np.zeros(outer + 1, dtype=np.int32)
    wits = np.zeros(cap + 1, dtype=np.int32)
    log = L.SolveLog(cap, *[a.ctypes.data_as(C.POINTER(C.c_double)) for a in bufs],
                     starts.ctypes.data_as(C.POINTER(C.c_int)), 0, 0, 0, 0, 0, 0, 0, 0,
                     wits.ctypes.data_as(C.POINTER(C.c_int)), 0)
    gt = None
    if opts.ground_truth is not None:
        gt = np.ascontiguousarray(np.asarray(opts.ground_truth), dtype=ndt).reshape(-1)
        pair.check_domain(gt.size)
    cb = L.OBSERVER()
    if opts.iterate_observer is not None:
        user = opts.iterate_observer

        def _obs(k, ptr, n, _u):
            arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float if t == "f32" else C.c_double)), shape=(n,))
            user(k, arr.copy())

        cb = L.OBSERVER(_obs)
    o = L.SolverOpts(opts.max_iters, int(opts.stop_on_explicit_residual_increase), opts.residual_tolerance,
                     int(opts.reorth), gt.ctypes.data_as(C.c_void_p) if gt is not None else None, cb, None)
    st = L.HybridStrategyC(int(strategy.kind), strategy.lambda_, strategy.noise_level) if strategy is not None else None
    sid = _SOLVER_ID[name]
    if dev:
        import torch

        x = torch.empty(pair.domain_size, dtype=b.dtype, device=b.device)
        torch.cuda.current_stream().synchronize()
        rc = getattr(lib, f"ctk_solve_dev_{t}")(proj.handle, sid, int(pair.variant), C.c_void_p(b.data_ptr()), lam,
                                                 C.byref(st) if st is not None else None, outer, inner, int(warm),
                                                 C.byref(o), C.c_void_p(x.data_ptr()), C.byref(log))
    else:
        bh = np.ascontiguousarray(np.asarray(b), dtype=ndt).reshape(-1)
        x = np.empty(pair.domain_size, dtype=ndt)
        bp, xp = bh.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p)
        v = int(pair.variant)
        if name in ("cgls", "lsqr", "sirt", "ab_gmres", "ba_gmres"):
            rc = getattr(lib, f"ctk_{name}_{t}")(proj.handle, v, bp, C.byref(o), xp, C.byref(log))
        elif name == "lsmr":
            rc = getattr(lib, f"ctk_lsmr_{t}")(proj.handle, v, bp, lam, C.byref(o), xp, C.byref(log))
        elif name in ("hybrid_lsqr", "flsqr_tv"):
            rc = getattr(lib, f"ctk_{name}_{t}")(proj.handle, v, bp, C.byref(st), C.byref(o), xp, C.byref(log))
        else:
            rc = getattr(lib, f"ctk_cgls_tv_{t}")(proj.handle, v, bp, lam, outer, inner, C.byref(o), int(warm), xp,
                                                   C.byref(log))
    _check(rc)
    it = log.iterations
    clog = ConvergenceLog(list(bufs[0][:it]), list(bufs[1][:it]), list(bufs[2][:log.n_relative_error]),
                          list(bufs[3][:log.n_lambda]), name, "single" if t == "f32" else "double", pair.matched)
    warnings = [f"tv preconditioner: inner CG not converged at iteration {int(k)}" for k in wits[:log.n_warnings]]
    return SolveResult(x, pair.domain_shape, log.iterations_run, StopReason(log.stop_reason), clog,
                       list(starts[:log.n_outer_starts]), log.stored_domain_basis, log.stored_range_basis, warnings)


def cgls(pair: OperatorPair, b, opts: SolverOptions) -> SolveResult:
    """solvers.hpp:13-60."""
    return _solve("cgls", pair, b, opts)


def lsqr(pair: OperatorPair, b, opts: SolverOptions) -> SolveResult:
    """solvers.hpp:62-126."""
    return _solve("lsqr", pair, b, opts)


def sirt(pair: OperatorPair, b, opts: SolverOptions) -> SolveResult:
    """solvers.hpp:233-287 (scaled Landweber with inverse row/column sums)."""
    return _solve("sirt", pair, b, opts)


def ab_gmres(pair: OperatorPair, b, opts: SolverOptions) -> SolveResult:
    """gmres.hpp:101-106: GMRES on min_u ||b - A B u||, x = B u."""
    return _solve("ab_gmres", pair, b, opts)


def ba_gmres(pair: OperatorPair, b, opts: SolverOptions) -> SolveResult:
    """gmres.hpp:108-113: GMRES on min_x ||B b - B A x||."""
    return _solve("ba_gmres", pair, b, opts)


def lsmr(pair: OperatorPair, b, lambda_: float, opts: SolverOptions) -> SolveResult:
    """solvers.hpp:128-231."""
    opts.validate()
    if lambda_ < 0.0:
        raise ParameterError("lsmr: lambda must be nonnegative")
    return _solve("lsmr", pair, b, opts, lam=lambda_)


def hybrid_lsqr(pair: OperatorPair, b, strategy: HybridStrategy, opts: SolverOptions) -> SolveResult:
    """hybrid.hpp:76-116."""
    return _solve("hybrid_lsqr", pair, b, opts, strategy=strategy)


def flsqr_tv(pair: OperatorPair, b, strategy: HybridStrategy, opts: SolverOptions) -> SolveResult:
    """tv.hpp:177-185: flexible hybrid LSQR with the TV priorconditioner (fixed or gcv)."""
    if strategy.kind == LambdaStrategy.dp:
        raise ParameterError("flsqr_tv: dp strategy is not supported, use fixed or gcv")
    return _solve("flsqr_tv", pair, b, opts, strategy=strategy)


def cgls_tv(pair: OperatorPair, b, lambda_: float, outer_iters: int, inner_iters: int, opts: SolverOptions,
            warm_start: bool = False) -> SolveResult:
    """tv.hpp:45-110."""
    return _solve("cgls_tv", pair, b, opts, lam=lambda_, outer=outer_iters, inner=inner_iters, warm=warm_start)


# ---- gradient, TV weights and operator compositions (gradient.hpp, tv.hpp:17-43,
#      operators.hpp:118-186) on the device ----------------------------------------------------
def _as_device(a, dtype=None):
    """(CUDA tensor, was_host) -- host arrays are copied to the device once."""
    import torch

    if _is_torch_cuda(a):
        t = a.reshape(-1)
        return (t.to(dtype) if dtype is not None and t.dtype != dtype else t).contiguous(), False
    h = np.ascontiguousarray(np.asarray(a)).reshape(-1)
    t = torch.from_numpy(h).cuda()
    return (t.to(dtype) if dtype is not None and t.dtype != dtype else t), True


def _like_input(t, was_host):
    return t.cpu().numpy() if was_host else t


def _vol_suffix(t):
    return Projector._suffix(t.dtype)


def gradient(vol, shape: VolumeShape):
    """gradient.hpp:9-30: forward differences (dx, dy, dz), zero on the far boundary."""
    import torch

    if shape.nx <= 0 or shape.ny <= 0 or shape.nz <= 0:
        raise DimensionError("volume dimensions must be positive")
    x, host = _as_device(vol)
    if x.numel() != shape.size():
        raise DimensionError("volume data length does not match nx*ny*nz")
    g = [torch.empty_like(x) for _ in range(3)]
    _check(getattr(L.load(), f"ctk_gradient_{_vol_suffix(x)}")(
        shape.nx, shape.ny, shape.nz, C.c_void_p(x.data_ptr()), *[C.c_void_p(v.data_ptr()) for v in g],
        _torch_stream()))
    return tuple(_like_input(v, host) for v in g)


def gradient_adjoint(dx, dy, dz, shape: VolumeShape):
    """gradient.hpp:32-54: the exact transpose of gradient()."""
    import torch

    comps = [_as_device(v) for v in (dx, dy, dz)]
    host = comps[0][1]
    g = [c[0] for c in comps]
    if any(v.numel() != shape.size() for v in g):
        raise DimensionError("gradient component lengths do not match volume shape")
    if len({v.dtype for v in g}) != 1:
        raise ParameterError("gradient components must share one dtype")
    out = torch.empty_like(g[0])
    _check(getattr(L.load(), f"ctk_gradient_adjoint_{_vol_suffix(out)}")(
        shape.nx, shape.ny, shape.nz, *[C.c_void_p(v.data_ptr()) for v in g], C.c_void_p(out.data_ptr()),
        _torch_stream()))
    return _like_input(out, host)


def tv_epsilon(x) -> float:
    """tv.hpp:17-24: 1e-4 * max|x|."""
    t, _ = _as_device(x)
    return 1e-4 * float(t.abs().max().double()) if t.numel() else 0.0


def tv_weights(x, shape: VolumeShape):
    """tv.hpp:26-43: w_i = (|Dx|_i^2 + eps^2)^(-1/4); all ones for an identically zero image."""
    import torch

    t, host = _as_device(x)
    if t.numel() != shape.size():
        raise DimensionError("volume data length does not match nx*ny*nz")
    eps = tv_epsilon(t)
    if eps == 0.0:
        return _like_input(torch.ones_like(t), host)
    w = torch.empty_like(t)
    _check(getattr(L.load(), f"ctk_tv_weights_{_vol_suffix(t)}")(shape.nx, shape.ny, shape.nz, C.c_void_p(t.data_ptr()),
                                                                eps, C.c_void_p(w.data_ptr()), _torch_stream()))
    return _like_input(w, host)


def _device_blas(name, t):
    return getattr(L.load(), f"ctk_{name}_{_vol_suffix(t)}")


def augment_tikhonov(pair: OperatorPair, lambda_: float) -> OperatorPair:
    """operators.hpp:118-139: forward x -> [A x; lambda x], back [y1; y2] -> B y1 + lambda y2."""
    if lambda_ < 0.0:
        raise ParameterError("tikhonov lambda must be nonnegative")
    nr, nd = pair.range_size, pair.domain_size

    def fwd(x, y):
        xd, host = _as_device(x)
        yd = _as_device(y)[0] if not host else __import__("torch").empty(nr + nd, dtype=xd.dtype, device="cuda")
        pair.forward(xd, yd[:nr])
        yd[nr:].copy_(xd)  # then y2 = T(lambda) * x in place
        _check(_device_blas("scal", xd)(nd, float(lambda_), C.c_void_p(yd[nr:].data_ptr()), _torch_stream()))
        if host:
            np.copyto(np.asarray(y).reshape(-1), yd.cpu().numpy())

    def bck(y, x):
        yd, host = _as_device(y)
        xd = _as_device(x)[0] if not host else __import__("torch").empty(nd, dtype=yd.dtype, device="cuda")
        pair.back(yd[:nr], xd)
        _check(_device_blas("axpy", yd)(nd, float(lambda_), C.c_void_p(yd[nr:].data_ptr()), C.c_void_p(xd.data_ptr()),
                                        _torch_stream()))
        if host:
            np.copyto(np.asarray(x).reshape(-1), xd.cpu().numpy())

    return OperatorPair(nd, nr + nd, pair.matched, pair.domain_shape, fwd, bck, pair.dtype, None, pair.variant)


def stack_weighted_gradient(pair: OperatorPair, lambda_: float, weights) -> OperatorPair:
    """operators.hpp:141-186: [A; lambda diag(w) D] -- range = measurements then the three
    weighted gradient components."""
    import torch

    nr, nd = pair.range_size, pair.domain_size
    w0, _ = _as_device(weights)
    if w0.numel() != nd:
        raise DimensionError("weight vector must have one entry per voxel")
    shape = pair.domain_shape

    def scaled(t):  # lambda * w in the operand's dtype (the reference forms lam * w[i] in T)
        w = w0.to(t.dtype)
        return w * torch.tensor(lambda_, dtype=t.dtype, device=w.device)

    def fwd(x, y):
        xd, host = _as_device(x)
        yd = _as_device(y)[0] if not host else torch.empty(nr + 3 * nd, dtype=xd.dtype, device="cuda")
        pair.forward(xd, yd[:nr])
        dx, dy, dz = gradient(xd, shape)
        s = scaled(xd)
        for q, comp in enumerate((dx, dy, dz)):
            yd[nr + q * nd: nr + (q + 1) * nd] = s * comp
        if host:
            np.copyto(np.asarray(y).reshape(-1), yd.cpu().numpy())

    def bck(y, x):
        yd, host = _as_device(y)
        xd = _as_device(x)[0] if not host else torch.empty(nd, dtype=yd.dtype, device="cuda")
        pair.back(yd[:nr], xd)
        s = scaled(yd)
        g = [s * yd[nr + q * nd: nr + (q + 1) * nd] for q in range(3)]
        xd += gradient_adjoint(*g, shape)
        if host:
            np.copyto(np.asarray(x).reshape(-1), xd.cpu().numpy())

    return OperatorPair(nd, nr + 3 * nd, pair.matched, shape, fwd, bck, pair.dtype, None, pair.variant)


# ---- synthetic input (phantom.hpp:118-145), generated on the device ---------------------------
def make_phantom(kind: PhantomKind, n: int, dtype="float32", device="cuda"):
    """make_phantom<T>(kind, n): shepp_logan_3d is n^3, the other two n*n*1 (x fastest).
    Bit-identical to the reference's rasteriser."""
    import torch

    kind = PhantomKind(kind)
    nz = n if kind == PhantomKind.shepp_logan_3d else 1
    t = torch.empty(max(n, 0) * max(n, 0) * nz, dtype=getattr(torch, dtype), device=device)
    suf = "f32" if dtype == "float32" else "f64"
    _check(getattr(L.load(), f"ctk_make_phantom_{suf}")(int(kind), n, C.c_void_p(t.data_ptr()), _torch_stream()))
    return t


def shepp_logan_3d(n: int, dtype="float32", device="cuda"):
    return make_phantom(PhantomKind.shepp_logan_3d, n, dtype, device)


# ---- measurement noise (noise.hpp:10-47) -------------------------------------------------------
@dataclass
class NoiseModel:
    """noise.hpp:12-22: air counts I0, electronic sigma (counts), RNG seed."""
    i0: float = 1e5
    sigma: float = 0.5
    seed: int = 0

    def validate(self):
        if not (self.i0 > 0.0):
            raise ParameterError("noise model: I0 must be positive")
        if self.sigma < 0.0:
            raise ParameterError("noise model: sigma must be nonnegative")


def noise_rng_id() -> str:
    """noise.hpp:24-27 (recorded in run metadata)."""
    return "mt19937_64+std::poisson/normal,sequential"


def add_noise(proj, model: NoiseModel):
    """add_noise<T> (noise.hpp:29-47) on a host array of line integrals -> a new array of
    the same dtype.  The single sequential mt19937_64 stream runs in libctk_b200.so on the
    host (the stream order is the definition; see csrc/noise.cpp)."""
    model.validate()
    a = np.asarray(proj)
    dt = np.float64 if a.dtype == np.float64 else np.float32
    src = np.ascontiguousarray(a, dtype=dt).reshape(-1)
    out = np.empty_like(src)
    fn = getattr(L.load(), "ctk_add_noise_" + ("f64" if dt == np.float64 else "f32"))
    _check(fn(src.size, src.ctypes.data_as(C.c_void_p), float(model.i0), float(model.sigma),
              int(model.seed) & 0xFFFFFFFFFFFFFFFF, out.ctypes.data_as(C.c_void_p)))
    return out


def launch_count() -> int:
    return int(L.load().ctk_launch_count())
