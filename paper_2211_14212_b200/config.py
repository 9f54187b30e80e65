"""Run configuration of the reconstruction pipeline (reference include/ctkrylov/config.hpp,
src/config.cpp): a flat ``key = value`` file, one pair per line, ``#`` comments, later keys
override earlier ones, unknown keys raise.  ``write_config`` serialises every field in the
reference's fixed order with the same number formatting, so files written here and by the
reference are byte-identical (tests/test_pipeline.py checks both directions).

Host-side text handling only; nothing here touches the GPU.
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass, field, fields
from typing import Dict, List, Optional

from .api import BeamMode, ParameterError, phantom_kind_from_string

_WS = " \t\n\v\f\r"  # std::isspace in the C locale (config.cpp:16-21)
_INT = re.compile(r"[ \t\n\v\f\r]*[+-]?[0-9]+\Z")
_DEC = re.compile(r"[ \t\n\v\f\r]*[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?\Z")
_HEX = re.compile(r"[ \t\n\v\f\r]*[+-]?0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?[0-9]+)?\Z")
_SPECIAL = re.compile(r"[ \t\n\v\f\r]*[+-]?(?:inf|infinity|nan(?:\([0-9A-Za-z_]*\))?)\Z", re.IGNORECASE)


def _trim(s: str) -> str:
    return s.strip(_WS)


def format_double(v: float) -> str:
    """%.17g (config.cpp:23-27)."""
    return "%.17g" % float(v)


def _parse_bool(v: str, key: str) -> bool:
    """config.cpp:29-33."""
    if v in ("true", "1", "yes", "on"):
        return True
    if v in ("false", "0", "no", "off"):
        return False
    raise ParameterError(f"config: boolean expected for {key}, got '{v}'")


def _parse_double(v: str, key: str) -> float:
    """std::stod with the whole string consumed (config.cpp:35-44); out-of-range values
    (overflow, or an underflow strtod flags) raise like std::out_of_range."""
    bad = ParameterError(f"config: number expected for {key}, got '{v}'")
    if _SPECIAL.match(v):
        t = v.strip(_WS).lower().lstrip("+-")
        sign = -1.0 if v.strip(_WS).startswith("-") else 1.0
        return sign * (math.inf if t.startswith("inf") else math.nan)
    if _DEC.match(v):
        d = float(v.strip(_WS))
    elif _HEX.match(v):
        d = float.fromhex(v.strip(_WS))
    else:
        raise bad
    mant = re.sub(r"[eEpP].*", "", v.strip(_WS).lstrip("+-"))
    mant = mant[2:] if mant[:2].lower() == "0x" else mant
    nonzero = any(c not in "0." for c in mant)
    if math.isinf(d) or (nonzero and abs(d) < 2.2250738585072014e-308):
        raise bad  # ERANGE -> std::out_of_range
    return d


def _parse_int(v: str, key: str) -> int:
    """std::stoll with the whole string consumed (config.cpp:46-55)."""
    if not _INT.match(v):
        raise ParameterError(f"config: integer expected for {key}, got '{v}'")
    d = int(v.strip(_WS))
    if not (-(1 << 63) <= d < (1 << 63)):
        raise ParameterError(f"config: integer expected for {key}, got '{v}'")
    return d


def _to_int32(d: int) -> int:
    """int(long long): two's-complement truncation, as gcc does."""
    d &= 0xFFFFFFFF
    return d - (1 << 32) if d >= (1 << 31) else d


def _split_list(v: str) -> List[str]:
    """std::getline on ',' with trimmed, non-empty items (config.cpp:57-66)."""
    parts = v.split(",")
    if parts and parts[-1] == "":
        parts.pop()  # getline yields no trailing empty item
    return [t for t in (_trim(p) for p in parts) if t]


@dataclass
class RunConfig:
    """config.hpp:18-70, same field names and defaults."""
    # phantom / data
    phantom: str = "shepp_logan_2d"
    size: int = 64
    # geometry
    geometry: str = "parallel2d"
    n_angles: int = 60
    angle_start_deg: float = 0.0
    angle_range_deg: float = 360.0
    detector_pixels_u: int = 0
    detector_pixels_v: int = 0
    detector_pixel_size: float = 0.0
    source_to_origin: float = 0.0
    origin_to_detector: float = 0.0
    spacing: float = 1.0
    # noise
    i0: float = 1e5
    sigma: float = 0.5
    seed: int = 0
    # solver
    solver: str = "lsqr"
    solvers: List[str] = field(default_factory=list)
    lambda_: float = 0.0
    strategy: str = "fixed"
    noise_level: float = 0.0
    outer_iters: int = 4
    inner_iters: int = 15
    warm_start: bool = False
    backprojector: str = "matched"
    max_iters: int = 30
    residual_tolerance: float = 1e-6
    stop_on_residual_increase: bool = True
    reorth: bool = True
    precision: str = "double"
    # io
    projections: str = ""
    ground_truth: str = ""
    output_dir: str = "."
    window_min: float = 0.0
    window_max: float = 0.0
    threads: int = 0

    def precision_kind(self) -> str:
        """config.cpp:70-74 -> "double" | "single"."""
        if self.precision in ("double", "single"):
            return self.precision
        raise ParameterError(f"config: precision must be single or double, got '{self.precision}'")

    def beam_mode(self) -> BeamMode:
        """config.cpp:76-81."""
        try:
            return BeamMode[self.geometry]
        except KeyError:
            raise ParameterError(f"config: unknown geometry '{self.geometry}'") from None

    def phantom_kind(self):
        return phantom_kind_from_string(self.phantom)

    def validate_common(self) -> None:
        """config.cpp:83-99, same checks in the same order."""
        self.phantom_kind()
        self.beam_mode()
        self.precision_kind()
        if self.size < 8:
            raise ParameterError("config: size must be at least 8")
        if self.n_angles < 1:
            raise ParameterError("config: n_angles must be at least 1")
        if self.max_iters < 1:
            raise ParameterError("config: max_iters must be at least 1")
        if self.residual_tolerance < 0:
            raise ParameterError("config: residual_tolerance must be >= 0")
        if not (self.i0 > 0):
            raise ParameterError("config: i0 must be positive")
        if self.sigma < 0:
            raise ParameterError("config: sigma must be >= 0")
        if self.lambda_ < 0:
            raise ParameterError("config: lambda must be >= 0")
        if self.threads < 0:
            raise ParameterError("config: threads must be >= 0")
        if self.backprojector not in ("matched", "voxel_driven"):
            raise ParameterError("config: backprojector must be matched or voxel_driven")
        if self.strategy not in ("fixed", "dp", "gcv"):
            raise ParameterError("config: strategy must be fixed, dp or gcv")

    def copy(self) -> "RunConfig":
        c = RunConfig(**{f.name: getattr(self, f.name) for f in fields(self)})
        c.solvers = list(self.solvers)
        return c


_STR = ("phantom", "geometry", "solver", "strategy", "backprojector", "precision", "projections",
        "ground_truth", "output_dir")
_INT32 = ("size", "n_angles", "detector_pixels_u", "detector_pixels_v", "outer_iters", "inner_iters",
          "max_iters", "threads")
_DBL = ("angle_start_deg", "angle_range_deg", "detector_pixel_size", "source_to_origin",
        "origin_to_detector", "spacing", "i0", "sigma", "lambda", "noise_level", "residual_tolerance",
        "window_min", "window_max")
_BOOL = ("warm_start", "stop_on_residual_increase", "reorth")


def apply_override(cfg: RunConfig, key: str, value: str) -> None:
    """One ``key=value`` assignment (config.cpp:101-138); unknown keys raise."""
    attr = "lambda_" if key == "lambda" else key
    if key in _STR:
        setattr(cfg, attr, value)
    elif key in _INT32:
        setattr(cfg, attr, _to_int32(_parse_int(value, key)))
    elif key in _DBL:
        setattr(cfg, attr, _parse_double(value, key))
    elif key in _BOOL:
        setattr(cfg, attr, _parse_bool(value, key))
    elif key == "seed":
        cfg.seed = _parse_int(value, key) & 0xFFFFFFFFFFFFFFFF  # std::uint64_t(long long)
    elif key == "solvers":
        cfg.solvers = _split_list(value)
    else:
        raise ParameterError(f"config: unknown key '{key}'")


def parse_config(text: str) -> RunConfig:
    """config.cpp:140-156."""
    cfg = RunConfig()
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for lineno, line in enumerate(lines, 1):
        hash_ = line.find("#")
        if hash_ >= 0:
            line = line[:hash_]
        line = _trim(line)
        if not line:
            continue
        eq = line.find("=")
        if eq < 0:
            raise ParameterError(f"config: line {lineno} has no '='")
        apply_override(cfg, _trim(line[:eq]), _trim(line[eq + 1:]))
    return cfg


def load_config(path) -> RunConfig:
    """config.cpp:158-162."""
    try:
        with open(path, "r", newline="") as f:
            text = f.read()
    except OSError:
        raise ParameterError(f"cannot open config: {path}") from None
    return parse_config(text)


def write_config(cfg: RunConfig, info: Optional[Dict[str, str]] = None) -> str:
    """config.cpp:164-210: ``# key: value`` info lines (sorted, as std::map), then every
    field in a fixed order.  Returns the text."""
    out = []
    for k in sorted(info or {}):
        out.append(f"# {k}: {info[k]}")
    c, g, b = cfg, format_double, (lambda v: "true" if v else "false")
    out += [f"phantom = {c.phantom}", f"size = {c.size}", f"geometry = {c.geometry}",
            f"n_angles = {c.n_angles}", f"angle_start_deg = {g(c.angle_start_deg)}",
            f"angle_range_deg = {g(c.angle_range_deg)}", f"detector_pixels_u = {c.detector_pixels_u}",
            f"detector_pixels_v = {c.detector_pixels_v}", f"detector_pixel_size = {g(c.detector_pixel_size)}",
            f"source_to_origin = {g(c.source_to_origin)}", f"origin_to_detector = {g(c.origin_to_detector)}",
            f"spacing = {g(c.spacing)}", f"i0 = {g(c.i0)}", f"sigma = {g(c.sigma)}", f"seed = {c.seed}",
            f"solver = {c.solver}"]
    if c.solvers:
        out.append("solvers = " + ",".join(c.solvers))
    out += [f"lambda = {g(c.lambda_)}", f"strategy = {c.strategy}", f"noise_level = {g(c.noise_level)}",
            f"outer_iters = {c.outer_iters}", f"inner_iters = {c.inner_iters}", f"warm_start = {b(c.warm_start)}",
            f"backprojector = {c.backprojector}", f"max_iters = {c.max_iters}",
            f"residual_tolerance = {g(c.residual_tolerance)}",
            f"stop_on_residual_increase = {b(c.stop_on_residual_increase)}", f"reorth = {b(c.reorth)}",
            f"precision = {c.precision}"]
    if c.projections:
        out.append(f"projections = {c.projections}")
    if c.ground_truth:
        out.append(f"ground_truth = {c.ground_truth}")
    out += [f"output_dir = {c.output_dir}", f"window_min = {g(c.window_min)}", f"window_max = {g(c.window_max)}",
            f"threads = {c.threads}"]
    return "\n".join(out) + "\n"
