"""Reconstruction metrics (reference include/ctkrylov/metrics.hpp).

``relative_residual`` is one genuine forward application plus two norms, on the device
through libctk_b200.so; ``relative_error`` is a device difference norm; the convergence-log
helpers and the CSV writer are host arithmetic on the (short) per-iteration histories.
Norms accumulate in fp64 on the device (the reference accumulates in T, so single-precision
values agree to f32 rounding, not bitwise).
"""
from __future__ import annotations

import ctypes as C
import io as _io
from dataclasses import dataclass

import numpy as np

from .api import (ConvergenceLog, DegenerateInputError, DimensionError, OperatorPair, ParameterError,
                  Projector, _check, _is_torch_cuda, _torch_stream)


def _device(a, dtype):
    import torch

    if _is_torch_cuda(a):
        return a.reshape(-1).to(dtype)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).reshape(-1))).to(device="cuda", dtype=dtype)


def _nrm2(lib, t, v) -> float:
    out = C.c_double()
    _check(getattr(lib, f"ctk_nrm2_{t}")(v.numel(), C.c_void_p(v.data_ptr()), C.byref(out), _torch_stream()))
    return out.value


def relative_residual(pair: OperatorPair, x, b) -> float:
    """||A x - b|| / ||b|| from one forward application (metrics.hpp:12-24)."""
    import torch

    pair.check_domain(x.numel() if _is_torch_cuda(x) else np.asarray(x).size)
    pair.check_range(b.numel() if _is_torch_cuda(b) else np.asarray(b).size)
    t = Projector._suffix(x.dtype)
    dt = torch.float32 if t == "f32" else torch.float64
    lib = pair.projector.lib
    xd, bd = _device(x, dt), _device(b, dt)
    bnorm = _nrm2(lib, t, bd)
    if not (bnorm > 0.0):
        raise DegenerateInputError("relative_residual: zero measurements")
    r = pair.apply_forward(xd)
    _check(getattr(lib, f"ctk_axpy_{t}")(r.numel(), -1.0, C.c_void_p(bd.data_ptr()), C.c_void_p(r.data_ptr()), _torch_stream()))
    return _nrm2(lib, t, r) / bnorm


def relative_error(x, gt, x_shape=None, gt_shape=None) -> float:
    """||x - gt|| / ||gt|| (metrics.hpp:26-36).  Shapes (VolumeShape) are compared when
    given, else the element counts."""
    import torch

    from . import _lib as L

    if (x_shape is not None and gt_shape is not None and x_shape != gt_shape) or \
            (x.numel() if _is_torch_cuda(x) else np.asarray(x).size) != \
            (gt.numel() if _is_torch_cuda(gt) else np.asarray(gt).size):
        raise DimensionError("relative_error: shape mismatch")
    src = x if _is_torch_cuda(x) else np.asarray(x)
    t = "f64" if src.dtype in (np.float64, torch.float64) else "f32"
    dt = torch.float32 if t == "f32" else torch.float64
    lib = L.load()
    xd, gd = _device(x, dt), _device(gt, dt)
    gnorm = _nrm2(lib, t, gd)
    if not (gnorm > 0.0):
        raise DegenerateInputError("relative_error: zero ground truth")
    d = xd.clone()
    _check(getattr(lib, f"ctk_axpy_{t}")(d.numel(), -1.0, C.c_void_p(gd.data_ptr()), C.c_void_p(d.data_ptr()), _torch_stream()))
    return _nrm2(lib, t, d) / gnorm


@dataclass
class Semiconvergence:
    """metrics.hpp:38-41."""
    min_index: int = 0
    rebound_ratio: float = 0.0


def detect_semiconvergence(log: ConvergenceLog) -> Semiconvergence:
    """First occurrence of the error minimum and the rebound after it (metrics.hpp:43-55)."""
    err = log.relative_error
    if len(err) < 3:
        raise ParameterError("detect_semiconvergence needs at least 3 error entries")
    best = 0
    for i in range(1, len(err)):
        if err[i] < err[best]:
            best = i
    return Semiconvergence(best, (err[-1] - err[best]) / err[best])


def residual_divergence(log: ConvergenceLog) -> float:
    """Worst relative gap between recurrence and explicit residuals (metrics.hpp:57-70)."""
    imp, exp = log.implicit_residual, log.explicit_residual
    if not imp or not exp or len(imp) != len(exp):
        raise ParameterError("residual_divergence needs both residual histories")
    worst = 0.0
    for a, b in zip(imp, exp):
        gap = abs(b - a) / max(a, 1e-30)
        worst = max(worst, gap)  # std::max keeps the first argument on NaN
    return worst


def csv_number(v: float) -> str:
    """%.12g (metrics.hpp:74-78)."""
    return "%.12g" % v


def write_csv(out, log: ConvergenceLog) -> None:
    """Fixed-layout convergence CSV (metrics.hpp:82-93): iter, implicit_residual,
    explicit_residual, relative_error, lambda; absent columns empty.  ``out`` is a path or
    a text stream."""
    buf = _io.StringIO()
    buf.write("iter,implicit_residual,explicit_residual,relative_error,lambda\n")
    cols = (log.implicit_residual, log.explicit_residual, log.relative_error, log.lambda_)
    for i in range(log.iterations()):
        buf.write(str(i + 1))
        for col in cols:
            buf.write("," + (csv_number(col[i]) if i < len(col) else ""))
        buf.write("\n")
    if isinstance(out, (str, bytes)) or hasattr(out, "__fspath__"):
        with open(out, "w", newline="") as f:
            f.write(buf.getvalue())
    else:
        out.write(buf.getvalue())


__all__ = ["relative_residual", "relative_error", "Semiconvergence", "detect_semiconvergence",
           "residual_divergence", "csv_number", "write_csv"]
