"""CPU tests of the drop-in boundary: libctk_b200.so loads without a GPU, exports every
entry point include/ctk_b200.h declares, and its host-side logic (geometry validation
with the reference's error taxonomy and messages, angle sharding, the projected-problem
helpers of hybrid LSQR) matches the reference -- no compute call needs a device here."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ctk_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctk_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import paper_2211_14212_b200 as ctk

    return ctk.load()


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("ctk_geom_create", "ctk_ax_f32", "ctk_atb_f32", "ctk_ax_f64", "ctk_atb_f64", "ctk_lsqr_f32",
                 "ctk_lsmr_f64", "ctk_hybrid_lsqr_f32", "ctk_cgls_tv_f64", "ctk_solve_dev_f32", "ctk_comm_create_nccl"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_abi_version(lib):
    assert lib.ctk_abi_version() == 2


def _desc(**kw):
    import paper_2211_14212_b200 as ctk

    g = ctk.bench_geometry(16, 8)
    for k, v in kw.items():
        if k in ("nx", "ny", "nz", "spacing"):
            setattr(g.vol, k, v)
        else:
            setattr(g, k, v)
    return g


@pytest.mark.parametrize("change,msg", [
    (dict(angles=[]), "geometry needs at least one angle"),
    (dict(nu=0), "detector pixel counts must be positive"),
    (dict(detector_pixel_size=0.0), "detector pixel size must be positive"),
    (dict(origin_to_detector=-1.0), "origin-to-detector distance must be positive"),
    (dict(nx=0), "geometry volume descriptor invalid"),
    (dict(source_to_origin=0.0), "cone3d requires a positive source-to-origin distance"),
    (dict(source_to_origin=5.0), "cone3d source lies inside the volume diagonal"),
])
def test_native_geometry_validation_mirrors_reference(lib, change, msg):
    """ConeGeometry::validate (geometry.hpp:35-54): same checks, order and wording, raised
    as GeometryError before any device work."""
    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200 import _lib as L

    g = _desc(**change)
    with pytest.raises(ctk.GeometryError, match=msg):
        g.validate()
    h = C.c_void_p()
    rc = lib.ctk_geom_create(C.byref(g.desc()), C.byref(h))
    assert rc == L.CTK_E_GEOMETRY
    assert L.last_error()[1] == msg


def test_parallel2d_requires_single_slice(lib):
    import paper_2211_14212_b200 as ctk

    g = ctk.ConeGeometry(ctk.BeamMode.parallel2d, 0.0, 8.0, 1.0, 12, 2, ctk.VolumeShape(8, 8, 1), [0.0])
    with pytest.raises(ctk.GeometryError, match="parallel2d requires nz = 1 and nv = 1"):
        ctk.Projector(g)


def test_reference_agrees_on_geometry_errors(reference):
    from oracle.oracle import RefError

    from geoms import cone_default

    g = cone_default(8, 4)
    g.dso = 5.0
    with pytest.raises(RefError) as e:
        reference.forward(g, np.zeros(g.domain_size))
    assert e.value.code == 2  # GeometryError


@pytest.mark.parametrize("na,G", [(360, 8), (360, 7), (10, 3), (5, 8), (1, 1), (720, 8)])
def test_shard_angles_partition(na, G):
    from paper_2211_14212_b200.comm import shard_angles

    blocks = [shard_angles(na, G, r) for r in range(G)]
    assert blocks[0][0] == 0
    for (f0, c0), (f1, c1) in zip(blocks, blocks[1:]):
        assert f0 + c0 == f1
    assert sum(c for _, c in blocks) == na
    assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1


def test_shard_angles_rejects_bad_input():
    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200.comm import shard_angles

    with pytest.raises(ctk.ParameterError):
        shard_angles(10, 2, 2)


def _bidiag(k, seed):
    rng = np.random.default_rng(seed)
    H = np.zeros((k + 1, k))
    for j in range(k):
        H[j, j] = 1.0 + rng.random()
        H[j + 1, j] = 0.5 * rng.random()
    return H


@pytest.mark.parametrize("k", [1, 2, 5, 12, 30])
def test_projected_helpers_vs_reference(lib, reference, k):
    """Host fp64 parameter choice of hybrid LSQR (regparam.hpp, hybrid.hpp:37-55) against the
    reference (Eigen-subset shim) and numpy."""
    from oracle.oracle import projected_tikhonov

    H = _bidiag(k, k)
    Hp = np.ascontiguousarray(H)
    p = Hp.ctypes.data_as(C.POINTER(C.c_double))
    out = C.c_double()
    assert lib.ctk_projected_gcv_lambda(p, k, 2.0, C.byref(out)) == 0
    assert out.value == pytest.approx(reference.gcv_lambda(H, 2.0), rel=1e-6)
    assert lib.ctk_projected_dp_lambda(p, k, 2.0, 0.05, C.byref(out)) == 0
    assert out.value == pytest.approx(reference.dp_lambda(H, 2.0, 0.05), rel=1e-6, abs=1e-14)
    y = np.zeros(k)
    fit = C.c_double()
    assert lib.ctk_projected_tikhonov(p, k, 2.0, 0.3, y.ctypes.data_as(C.POINTER(C.c_double)), C.byref(fit)) == 0
    yw, fw = projected_tikhonov(H, 2.0, 0.3)
    assert np.allclose(y, yw, rtol=1e-10, atol=1e-13)
    assert fit.value == pytest.approx(fw, rel=1e-10)


def test_dp_rejects_bad_noise_level(lib):
    H = np.ascontiguousarray(_bidiag(3, 1))
    out = C.c_double()
    assert lib.ctk_projected_dp_lambda(H.ctypes.data_as(C.POINTER(C.c_double)), 3, 1.0, 1.5, C.byref(out)) == 3


def test_python_mirror_surface():
    """The host mirror exposes the reference's public names (api.py docstring map)."""
    import paper_2211_14212_b200 as ctk

    for name in ("ConeGeometry", "BeamMode", "BackprojectVariant", "OperatorPair", "projector_pair",
                 "forward_project", "back_project", "SolverOptions", "SolveResult", "cgls", "lsqr", "lsmr",
                 "hybrid_lsqr", "cgls_tv", "HybridStrategy", "equidistant_angles", "default_geometry",
                 "DimensionError", "GeometryError", "ParameterError", "DegenerateInputError", "NumericalError"):
        assert hasattr(ctk, name), name
    g = ctk.default_geometry(ctk.BeamMode.cone3d, ctk.VolumeShape(16, 16, 16), 10)
    assert (g.nu, g.nv, g.source_to_origin, g.origin_to_detector, g.detector_pixel_size) == (24, 24, 32.0, 16.0, 1.5)
    assert ctk.equidistant_angles(4) == [0.0, math.pi / 2, math.pi, 3 * math.pi / 2]
    with pytest.raises(ctk.ParameterError):
        ctk.HybridStrategy.dp(1.5)
    with pytest.raises(ctk.ParameterError):
        ctk.SolverOptions(max_iters=0).validate()
