"""The pybind11 `_core` module (the reference's module name, bindings/bindings.cpp:1-2) on the
CPU: it imports, exposes the reference's names, and its host-side logic (geometry defaults
and validation, strategy checks) agrees with the ctypes mirror (api.py)."""
import numpy as np
import pytest

import paper_2211_14212_b200 as ctk
from paper_2211_14212_b200 import _core


def test_core_exports_reference_names():
    for name in ("BeamMode", "BackprojectVariant", "ProjectorKind", "StopReason", "VolumeShape", "ConeGeometry",
                 "default_geometry", "equidistant_angles", "canonical_angle", "projector_pair", "OperatorPair",
                 "SolverOptions", "SolveResult", "ConvergenceLog", "HybridStrategy", "cgls", "lsqr", "lsmr", "sirt",
                 "hybrid_lsqr", "cgls_tv", "flsqr_tv", "ab_gmres", "ba_gmres", "DimensionError", "GeometryError",
                 "ParameterError", "DegenerateInputError", "NumericalError"):
        assert hasattr(_core, name), name
    assert _core.abi_version == ctk.load().ctk_abi_version()


@pytest.mark.parametrize("mode", ["parallel2d", "parallel3d", "cone3d"])
def test_default_geometry_matches_mirror(mode):
    nz = 1 if mode == "parallel2d" else 20
    g = _core.default_geometry(getattr(_core.BeamMode, mode), _core.VolumeShape(24, 22, nz, 0.7), 17, 3.0)
    w = ctk.default_geometry(getattr(ctk.BeamMode, mode), ctk.VolumeShape(24, 22, nz, 0.7), 17, 3.0)
    assert (g.nu, g.nv, g.source_to_origin, g.origin_to_detector, g.detector_pixel_size) == \
        (w.nu, w.nv, w.source_to_origin, w.origin_to_detector, w.detector_pixel_size)
    assert np.array_equal(np.asarray(g.angles), np.asarray(w.angles, dtype=np.float64))
    assert _core.canonical_angle(-1.0) == ctk.canonical_angle(-1.0)


def _both_raise(mutate):
    g = _core.default_geometry(_core.BeamMode.cone3d, _core.VolumeShape(16, 16, 16), 8)
    w = ctk.default_geometry(ctk.BeamMode.cone3d, ctk.VolumeShape(16, 16, 16), 8)
    mutate(g)
    mutate(w)
    with pytest.raises(_core.GeometryError) as e1:
        g.validate()
    with pytest.raises(ctk.GeometryError) as e2:
        w.validate()
    assert str(e1.value) == str(e2.value)


@pytest.mark.parametrize("field,value", [("nu", 0), ("detector_pixel_size", 0.0), ("origin_to_detector", -1.0),
                                         ("source_to_origin", 5.0), ("angles", [])])
def test_validation_messages_match_mirror(field, value):
    _both_raise(lambda g: setattr(g, field, value))


def test_strategy_and_option_errors():
    with pytest.raises(_core.ParameterError, match="dp strategy needs a noise level"):
        _core.HybridStrategy.dp(1.5)
    with pytest.raises(_core.ParameterError, match="fixed lambda must be nonnegative"):
        _core.HybridStrategy.fixed(-1.0)
    with pytest.raises(_core.ParameterError, match="max_iters must be >= 1"):
        _core.SolverOptions(max_iters=0).validate()
    with pytest.raises(_core.GeometryError, match="angle count must be positive"):
        _core.equidistant_angles(0)
    assert issubclass(_core.NumericalError, _core.CtkError) and issubclass(_core.CtkError, RuntimeError)
