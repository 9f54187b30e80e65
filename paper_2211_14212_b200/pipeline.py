"""The reconstruction pipeline around the hot path (reference include/ctkrylov/pipeline.hpp,
src/pipeline.cpp): ``run_simulate`` (phantom -> clean projections -> count-domain noise),
``run_reconstruct`` (one solver on a projection file) and ``run_compare`` (several solvers on
identical data), writing the reference's files with the reference's names and formats.

Every operator application and solve runs through the device path (``projector_pair`` +
the device solvers; double precision selects the exact-parity f64 kernels, so a double
``run_simulate`` writes byte-identical files to the reference's).  The host does the file
I/O, the sequential noise stream (csrc/noise.cpp) and the bookkeeping.
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

from . import io as cio
from .api import (BackprojectVariant, ConeGeometry, ConvergenceLog, DimensionError, HybridStrategy,
                  NoiseModel, ParameterError, PhantomKind, SolveResult, SolverOptions, VolumeShape, ab_gmres,
                  add_noise, ba_gmres, canonical_angle, cgls, cgls_tv, default_geometry, equidistant_angles,
                  flsqr_tv, hybrid_lsqr, lsmr, lsqr, make_phantom, noise_rng_id, projector_pair, sirt)
from .config import RunConfig, write_config
from .metrics import csv_number, write_csv

_DEG2RAD = math.pi / 180.0  # pipeline.cpp:28


def _phantom_shape(cfg: RunConfig) -> VolumeShape:
    """pipeline.cpp:38-42."""
    n = cfg.size
    flat = cfg.phantom_kind() != PhantomKind.shepp_logan_3d
    return VolumeShape(n, n, 1 if flat else n, cfg.spacing)


def _ensure_output_dir(cfg: RunConfig) -> None:
    """pipeline.cpp:44-48."""
    try:
        os.makedirs(cfg.output_dir, exist_ok=True)
    except OSError:
        pass
    if not os.path.isdir(cfg.output_dir):
        raise ParameterError("output directory is not writable: " + cfg.output_dir)


def _write_metadata(path: str, cfg: RunConfig, info: Dict[str, str]) -> None:
    """pipeline.cpp:50-56."""
    info = dict(info)
    info["rng"] = noise_rng_id()
    try:
        with open(path, "w", newline="") as f:
            f.write(write_config(cfg, info))
    except OSError:
        raise ParameterError("cannot write metadata: " + path) from None


def _std_to_string(v: float) -> str:
    """std::to_string(double) is "%f"."""
    return "%f" % v


def solver_label(cfg: RunConfig, name: str) -> str:
    """pipeline.cpp:58-62."""
    if name == "lsmr":
        return f"{name}(lambda={_std_to_string(cfg.lambda_)})"
    if name in ("hybrid_lsqr", "flsqr_tv"):
        return f"{name}({cfg.strategy})"
    return name


def _strategy_from(cfg: RunConfig) -> HybridStrategy:
    """pipeline.cpp:64-68."""
    if cfg.strategy == "fixed":
        return HybridStrategy.fixed(cfg.lambda_)
    if cfg.strategy == "dp":
        return HybridStrategy.dp(cfg.noise_level)
    return HybridStrategy.gcv()


def _options_from(cfg: RunConfig, gt: Optional[np.ndarray], dtype) -> SolverOptions:
    """pipeline.cpp:70-81."""
    return SolverOptions(max_iters=cfg.max_iters, stop_on_explicit_residual_increase=cfg.stop_on_residual_increase,
                         residual_tolerance=cfg.residual_tolerance, reorth=cfg.reorth,
                         ground_truth=None if gt is None else gt.astype(dtype), rng_seed=cfg.seed)


def run_named_solver(name: str, pair, b, cfg: RunConfig, opts: SolverOptions) -> SolveResult:
    """pipeline.cpp:83-101."""
    if name == "cgls":
        return cgls(pair, b, opts)
    if name == "lsqr":
        return lsqr(pair, b, opts)
    if name == "lsmr":
        return lsmr(pair, b, cfg.lambda_, opts)
    if name == "sirt":
        return sirt(pair, b, opts)
    if name == "ab_gmres":
        return ab_gmres(pair, b, opts)
    if name == "ba_gmres":
        return ba_gmres(pair, b, opts)
    if name == "hybrid_lsqr":
        return hybrid_lsqr(pair, b, _strategy_from(cfg), opts)
    if name == "cgls_tv":
        return cgls_tv(pair, b, cfg.lambda_, cfg.outer_iters, cfg.inner_iters, opts, cfg.warm_start)
    if name == "flsqr_tv":
        return flsqr_tv(pair, b, _strategy_from(cfg), opts)
    raise ParameterError("unknown solver: " + name)


def export_slices(directory: str, vol: np.ndarray, shape: VolumeShape, wmin: float, wmax: float) -> None:
    """Central transversal (fixed z, nx x ny) and sagittal (fixed x, ny x nz) 16-bit PGMs
    (pipeline.cpp:103-129); an empty window [wmin >= wmax] means the data's min/max."""
    v = np.asarray(vol, dtype=np.float32).reshape(shape.nz, shape.ny, shape.nx)
    if wmax <= wmin:
        wmin = float(v.min()) if v.size else 0.0
        wmax = float(v.max()) if v.size else 1.0
    k = shape.nz // 2
    cio.write_pgm16(os.path.join(directory, "slice_transversal.pgm"), shape.nx, shape.ny, v[k].reshape(-1), wmin, wmax)
    i = shape.nx // 2
    cio.write_pgm16(os.path.join(directory, "slice_sagittal.pgm"), shape.ny, shape.nz,
                    np.ascontiguousarray(v[:, :, i]).reshape(-1), wmin, wmax)


def resolve_geometry(cfg: RunConfig) -> ConeGeometry:
    """pipeline.cpp:241-262: auto (zero) geometry fields resolved in place to the
    desk-scale defaults; returns the acquisition the run uses."""
    cfg.validate_common()
    vol = _phantom_shape(cfg)
    g = default_geometry(cfg.beam_mode(), vol, cfg.n_angles, cfg.angle_range_deg * _DEG2RAD)
    g.angles = equidistant_angles(cfg.n_angles, cfg.angle_start_deg * _DEG2RAD, cfg.angle_range_deg * _DEG2RAD)
    if cfg.detector_pixels_u > 0:
        g.nu = cfg.detector_pixels_u
    if cfg.detector_pixels_v > 0:
        g.nv = cfg.detector_pixels_v
    if cfg.detector_pixel_size > 0:
        g.detector_pixel_size = cfg.detector_pixel_size
    if cfg.source_to_origin > 0:
        g.source_to_origin = cfg.source_to_origin
    if cfg.origin_to_detector > 0:
        g.origin_to_detector = cfg.origin_to_detector
    g.validate()
    cfg.detector_pixels_u, cfg.detector_pixels_v = g.nu, g.nv
    cfg.detector_pixel_size = g.detector_pixel_size
    cfg.source_to_origin, cfg.origin_to_detector = g.source_to_origin, g.origin_to_detector
    return g


def run_simulate(cfg: RunConfig) -> None:
    """pipeline.cpp:264-289: phantom.vol, projections_clean.proj, projections_noisy.proj,
    simulate_meta.cfg (itself a config reproducing the run)."""
    import torch

    cfg = cfg.copy()
    _ensure_output_dir(cfg)
    geom = resolve_geometry(cfg)
    n = cfg.size
    phantom = make_phantom(cfg.phantom_kind(), n, "float32")  # make_phantom<float>, spacing 1.0
    pshape = VolumeShape(n, n, n if cfg.phantom_kind() == PhantomKind.shepp_logan_3d else 1, 1.0)
    if pshape != geom.vol:
        raise DimensionError("volume shape does not match geometry descriptor")  # projector.hpp:138
    if cfg.precision_kind() == "double":
        pair = projector_pair(geom, dtype=np.float64)
        clean = pair.apply_forward(phantom.double()).float()  # projections_from(forward_project<double>)
    else:
        pair = projector_pair(geom)
        clean = pair.apply_forward(phantom)
    clean_h = clean.cpu().numpy()
    torch.cuda.synchronize()
    angles = [canonical_angle(a) for a in geom.angles]
    noisy = add_noise(clean_h, NoiseModel(cfg.i0, cfg.sigma, cfg.seed))
    d = cfg.output_dir
    cio.save_volume(os.path.join(d, "phantom.vol"), phantom.cpu().numpy(), pshape)
    cio.save_projections(os.path.join(d, "projections_clean.proj"), clean_h, angles, geom.nu, geom.nv)
    cio.save_projections(os.path.join(d, "projections_noisy.proj"), noisy, angles, geom.nu, geom.nv)
    cfg.projections = os.path.join(d, "projections_noisy.proj")
    cfg.ground_truth = os.path.join(d, "phantom.vol")
    _write_metadata(os.path.join(d, "simulate_meta.cfg"), cfg, {"command": "simulate"})


@dataclass
class RunSummary:
    """pipeline.cpp:160-171."""
    label: str = ""
    iterations: int = 0
    stop_reason: str = ""
    min_error: float = math.nan
    min_error_iter: int = -1
    rebound_ratio: float = math.nan
    final_residual: float = math.nan
    wall_seconds: float = 0.0
    log: Optional[ConvergenceLog] = None


def _summarize(label: str, res: SolveResult, secs: float) -> RunSummary:
    """pipeline.cpp:173-193."""
    s = RunSummary(label, res.iterations_run, res.stop_reason.name, wall_seconds=secs, log=res.log)
    if res.log.explicit_residual:
        s.final_residual = res.log.explicit_residual[-1]
    err = res.log.relative_error
    if err:
        best = 0
        for i in range(1, len(err)):
            if err[i] < err[best]:
                best = i
        s.min_error, s.min_error_iter = err[best], best + 1
        s.rebound_ratio = (err[-1] - err[best]) / err[best]
    return s


def _geometry_for_data(cfg: RunConfig, angles, nu: int, nv: int) -> ConeGeometry:
    """pipeline.cpp:133-141: distances and pixel size from the config, angles and detector
    counts from the projection file."""
    g = resolve_geometry(cfg)
    g.angles, g.nu, g.nv = list(angles), nu, nv
    g.validate()
    return g


def _execute(name: str, cfg: RunConfig, proj, gt, want_recon: bool):
    """execute_one / execute_dispatch (pipeline.cpp:195-219); cfg is taken by value."""
    cfg = cfg.copy()
    cfg.solver = name
    data, angles, nu, nv = proj
    dt = np.float64 if cfg.precision_kind() == "double" else np.float32
    geom = _geometry_for_data(cfg, angles, nu, nv)
    variant = BackprojectVariant.matched if cfg.backprojector == "matched" else BackprojectVariant.voxel_driven
    pair = projector_pair(geom, variant, dtype=dt)
    b = np.ascontiguousarray(data, dtype=dt)
    opts = _options_from(cfg, gt, dt)
    t0 = time.perf_counter()
    res = run_named_solver(name, pair, b, cfg, opts)
    secs = time.perf_counter() - t0
    recon = np.asarray(res.x, dtype=np.float32) if want_recon else None  # volume_from<T>
    return _summarize(solver_label(cfg, name), res, secs), recon, pair.domain_shape


def _load_inputs(cfg: RunConfig):
    proj = cio.load_projections(cfg.projections)
    gt = None
    if cfg.ground_truth:
        gt, _ = cio.load_volume(cfg.ground_truth)
    return proj, gt


def _fmt_g(v: float) -> str:
    return "%.6g" % v


def run_reconstruct(cfg: RunConfig) -> RunSummary:
    """pipeline.cpp:291-316: recon.vol, two central PGM slices, convergence.csv,
    reconstruct_meta.cfg."""
    cfg = cfg.copy()
    cfg.validate_common()
    if not cfg.projections:
        raise ParameterError("reconstruct needs a projections file (projections = PATH)")
    _ensure_output_dir(cfg)
    proj, gt = _load_inputs(cfg)
    s, recon, shape = _execute(cfg.solver, cfg, proj, gt, True)
    d = cfg.output_dir
    cio.save_volume(os.path.join(d, "recon.vol"), recon, shape)
    export_slices(d, recon, shape, cfg.window_min, cfg.window_max)
    write_csv(os.path.join(d, "convergence.csv"), s.log)
    _write_metadata(os.path.join(d, "reconstruct_meta.cfg"), cfg,
                    {"command": "reconstruct", "stop_reason": s.stop_reason, "iterations": str(s.iterations),
                     "wall_seconds": _fmt_g(s.wall_seconds)})
    return s


def run_compare(cfg: RunConfig) -> List[RunSummary]:
    """pipeline.cpp:318-351: per-solver CSVs, compare_wide.csv, summary.txt,
    compare_meta.cfg."""
    cfg = cfg.copy()
    cfg.validate_common()
    if len(cfg.solvers) < 2:
        raise ParameterError("compare needs at least two solvers (solvers = a,b,...)")
    if not cfg.projections:
        raise ParameterError("compare needs a projections file (projections = PATH)")
    _ensure_output_dir(cfg)
    proj, gt = _load_inputs(cfg)
    d = cfg.output_dir
    rows = []
    for name in cfg.solvers:
        s, _, _ = _execute(name, cfg, proj, gt, False)
        write_csv(os.path.join(d, name + ".csv"), s.log)
        rows.append(s)

    def cell(v, i):
        return csv_number(v[i]) if i < len(v) else ""

    out = ["iter" + "".join(f",{r.label}.{c}" for r in rows
                            for c in ("implicit_residual", "explicit_residual", "relative_error", "lambda"))]
    for i in range(max(r.log.iterations() for r in rows)):
        out.append(str(i + 1) + "".join(
            f",{cell(r.log.implicit_residual, i)},{cell(r.log.explicit_residual, i)},"
            f"{cell(r.log.relative_error, i)},{cell(r.log.lambda_, i)}" for r in rows))
    with open(os.path.join(d, "compare_wide.csv"), "w", newline="") as f:
        f.write("\n".join(out) + "\n")
    lines = ["solver  iterations  stop_reason  min_rel_error  min_error_iter  "
             "rebound_ratio  final_explicit_residual  wall_seconds"]
    for r in rows:
        lines.append(f"{r.label}  {r.iterations}  {r.stop_reason}  {_fmt_g(r.min_error)}  {r.min_error_iter}  "
                     f"{_fmt_g(r.rebound_ratio)}  {_fmt_g(r.final_residual)}  {_fmt_g(r.wall_seconds)}")
    with open(os.path.join(d, "summary.txt"), "w", newline="") as f:
        f.write("\n".join(lines) + "\n")
    _write_metadata(os.path.join(d, "compare_meta.cfg"), cfg, {"command": "compare"})
    return rows


__all__ = ["resolve_geometry", "run_simulate", "run_reconstruct", "run_compare", "export_slices", "solver_label",
           "run_named_solver", "RunSummary"]
