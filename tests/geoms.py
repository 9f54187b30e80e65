"""Shared test geometries (oracle Geom <-> product ConeGeometry)."""
import math

import numpy as np

from oracle.oracle import CONE3D, PARALLEL2D, PARALLEL3D, Geom, equidistant_angles


def to_ctk(g: Geom):
    import paper_2211_14212_b200 as ctk

    return ctk.ConeGeometry(ctk.BeamMode(g.mode), g.dso, g.dod, g.du, g.nu, g.nv,
                            ctk.VolumeShape(g.nx, g.ny, g.nz, g.h), list(np.asarray(g.angles, dtype=np.float64)))


def parallel2d(n=32, na=24, nu=None):
    # test_operators.cpp:13-23
    return Geom(PARALLEL2D, 0.0, float(n), 1.0, nu or (3 * n) // 2, 1, n, n, 1, 1.0, equidistant_angles(na))


def parallel3d(nx=16, ny=14, nz=8, na=10):
    return Geom(PARALLEL3D, 0.0, 16.0, 1.0, 24, 12, nx, ny, nz, 1.0, equidistant_angles(na))


def cone_default(n=24, na=18):
    # default_geometry(cone3d) (geometry.hpp:74-78): DSO 2n, DOD n, pixel 1.5, nu = nv = 3n/2
    return Geom(CONE3D, 2.0 * n, 1.0 * n, 1.5, (3 * n) // 2, (3 * n) // 2, n, n, n, 1.0, equidistant_angles(na))


def cone_bench(n=64, na=100):
    # the configs' geometry: nu = nv = n
    return Geom(CONE3D, 2.0 * n, 1.0 * n, 1.5, n, n, n, n, n, 1.0, equidistant_angles(na))


def cone_ragged():
    # odd, non-cubic volume, non-square detector, angles off the equidistant grid, h != 1
    ang = np.sort(np.array([0.0, 0.3, 0.7853981633974483, 1.1, 2.0, 2.356194490192345, 3.9, 5.5]))
    return Geom(CONE3D, 40.0, 25.0, 1.2, 23, 17, 20, 13, 7, 0.9, ang)


def cone_steep():
    # tall detector close to the source: many rays are z-dominant (generic path)
    n = 16
    return Geom(CONE3D, 14.5, 30.0, 2.0, 12, 64, n, n, n, 1.0, equidistant_angles(6))


def cone_adjoint():
    # test_operators.cpp:177-188
    return Geom(CONE3D, 30.0, 12.0, 1.5, 18, 18, 12, 12, 12, 1.0, equidistant_angles(9))


def cone_multitile():
    # rows per plane (140, 300) span several 128-row tiles of the f32 plane backprojector with
    # ragged ends; 40 slices = a full and a ragged 32-slice band
    return Geom(CONE3D, 400.0, 200.0, 2.5, 200, 32, 300, 140, 40, 1.0, equidistant_angles(24))


def cone_wide():
    # 800 rows per plane in the y-dominant pass: the 256-row tiles of the plane backprojector
    return Geom(CONE3D, 900.0, 300.0, 4.0, 300, 8, 800, 24, 8, 1.0, equidistant_angles(20))


ALL = {
    "parallel2d": parallel2d,
    "parallel3d": parallel3d,
    "cone_default": cone_default,
    "cone_ragged": cone_ragged,
    "cone_steep": cone_steep,
    "cone_adjoint": cone_adjoint,
    "cone_multitile": cone_multitile,
    "cone_wide": cone_wide,
}
