"""On-disk formats around the path (reference src/io.cpp:1-120,
include/ctkrylov/io.hpp): 32-bit little-endian raw floats with a text sidecar
``<path>.hdr``, and the 16-bit binary PGM preview.

  volume       raw x[i + nx(j + ny k)], header "nx ny nz spacing" (spacing %.17g)
  projections  raw y[iu + nu(iv + nv a)], header "n_angles nu nv" then one angle per line

Byte-for-byte the reference's files (tests/test_io.py writes with one side and reads with
the other).  Host-side byte work: nothing here touches the GPU.
"""
from __future__ import annotations

import os
import sys

import numpy as np

from .api import DimensionError, ParameterError, VolumeShape

if sys.byteorder != "little":  # io.cpp:9-10
    raise ImportError("raw file formats assume a little-endian host")


def _hdr(path) -> str:
    return os.fspath(path) + ".hdr"


def _g17(v: float) -> str:
    return "%.17g" % float(v)  # format_double, io.cpp:40-44


def _write_raw(path, data: np.ndarray) -> None:
    try:
        with open(path, "wb") as f:
            f.write(np.ascontiguousarray(data, dtype="<f4").tobytes())
    except OSError as e:
        raise ParameterError(f"cannot open for writing: {os.fspath(path)}") from e


def _read_raw(path, n: int) -> np.ndarray:
    try:
        with open(path, "rb") as f:
            raw = f.read(4 * n)
    except OSError as e:
        raise ParameterError(f"cannot open for reading: {os.fspath(path)}") from e
    if len(raw) != 4 * n:
        raise DimensionError(f"raw file shorter than its header promises: {os.fspath(path)}")
    return np.frombuffer(raw, dtype="<f4").astype(np.float32)


def _read_header(path):
    try:
        with open(_hdr(path), "r") as h:
            return h.read().split()
    except OSError as e:
        raise ParameterError(f"missing header: {_hdr(path)}") from e


def save_volume(path, data, shape: VolumeShape) -> None:
    """io.cpp:48-54 (Volume::validate first: the data must hold nx*ny*nz values)."""
    a = np.asarray(data, dtype=np.float32).reshape(-1)
    if shape.nx <= 0 or shape.ny <= 0 or shape.nz <= 0 or a.size != shape.size():
        raise DimensionError("volume data does not match its shape")
    _write_raw(path, a)
    try:
        with open(_hdr(path), "w") as h:
            h.write(f"{shape.nx} {shape.ny} {shape.nz} {_g17(shape.spacing)}\n")
    except OSError as e:
        raise ParameterError(f"cannot open for writing: {_hdr(path)}") from e


def load_volume(path):
    """io.cpp:56-66 -> (data [nx*ny*nz] float32, VolumeShape)."""
    tok = _read_header(path)
    try:
        nx, ny, nz, spacing = int(tok[0]), int(tok[1]), int(tok[2]), float(tok[3])
    except (IndexError, ValueError) as e:
        raise ParameterError(f"malformed volume header: {_hdr(path)}") from e
    shape = VolumeShape(nx, ny, nz, spacing)
    if nx <= 0 or ny <= 0 or nz <= 0:
        raise DimensionError("volume dimensions must be positive")
    return _read_raw(path, shape.size()), shape


def save_projections(path, data, angles, nu: int, nv: int) -> None:
    """io.cpp:68-75: header "n_angles nu nv" then one angle (%.17g) per line."""
    a = np.asarray(data, dtype=np.float32).reshape(-1)
    angles = [float(x) for x in angles]
    if nu <= 0 or nv <= 0 or a.size != len(angles) * nu * nv:
        raise DimensionError("projection data does not match its shape")
    _write_raw(path, a)
    try:
        with open(_hdr(path), "w") as h:
            h.write(f"{len(angles)} {nu} {nv}\n")
            for x in angles:
                h.write(_g17(x) + "\n")
    except OSError as e:
        raise ParameterError(f"cannot open for writing: {_hdr(path)}") from e


def load_projections(path):
    """io.cpp:77-90 -> (data [n_angles*nv*nu] float32, angles, nu, nv)."""
    tok = _read_header(path)
    try:
        na, nu, nv = int(tok[0]), int(tok[1]), int(tok[2])
    except (IndexError, ValueError) as e:
        raise ParameterError(f"malformed projection header: {_hdr(path)}") from e
    na = max(na, 0)
    try:
        angles = [float(t) for t in tok[3:3 + na]]
    except ValueError as e:
        raise ParameterError("projection header is missing angles") from e
    if len(angles) != na:
        raise ParameterError("projection header is missing angles")
    if nu <= 0 or nv <= 0:
        raise DimensionError("projection dimensions must be positive")
    return _read_raw(path, na * nu * nv), angles, nu, nv


def write_pgm16(path, width: int, height: int, values, wmin: float, wmax: float) -> None:
    """io.cpp:92-116: P5, maxval 65535, big-endian samples, window [wmin, wmax] clamped."""
    if width <= 0 or height <= 0:
        raise DimensionError("pgm dimensions must be positive")
    if not wmax > wmin:
        wmax = wmin + 1.0
    v = np.asarray(values, dtype=np.float32).reshape(-1)[: width * height].astype(np.float64)
    scale = 65535.0 / (wmax - wmin)
    q = (np.clip((v - wmin) * scale, 0.0, 65535.0) + 0.5).astype(np.uint32)
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{width} {height}\n65535\n".encode())
            f.write(q.astype(">u2").tobytes())
    except OSError as e:
        raise ParameterError(f"cannot open for writing: {os.fspath(path)}") from e
