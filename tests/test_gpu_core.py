"""The pybind11 `_core` against the ctypes mirror on the GPU: same native entry points, so
operators and solvers must agree bit for bit."""
import numpy as np
import pytest

import paper_2211_14212_b200 as ctk
from paper_2211_14212_b200 import _core

pytestmark = pytest.mark.gpu


def _geoms(n=20, na=12):
    g = _core.default_geometry(_core.BeamMode.cone3d, _core.VolumeShape(n, n, n), na)
    w = ctk.default_geometry(ctk.BeamMode.cone3d, ctk.VolumeShape(n, n, n), na)
    return g, w


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("variant", ["matched", "voxel_driven"])
def test_core_operators_bitwise(dtype, variant):
    g, w = _geoms()
    pc = _core.projector_pair(g, getattr(_core.BackprojectVariant, variant), np.dtype(dtype).name)
    pw = ctk.projector_pair(w, getattr(ctk.BackprojectVariant, variant), dtype)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(pc.domain_size).astype(dtype)
    y = rng.standard_normal(pc.range_size).astype(dtype)
    assert pc.domain_size == pw.domain_size and pc.range_size == pw.range_size
    assert np.array_equal(pc.apply_forward(x), pw.apply_forward(x))
    assert np.array_equal(pc.apply_back(y), pw.apply_back(y))
    with pytest.raises(_core.DimensionError, match="operator domain size mismatch"):
        pc.apply_forward(x[:-1])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_core_solvers_bitwise(dtype):
    g, w = _geoms()
    pc = _core.projector_pair(g, _core.BackprojectVariant.matched, np.dtype(dtype).name)
    pw = ctk.projector_pair(w, ctk.BackprojectVariant.matched, dtype)
    x_true = ctk.shepp_logan_3d(20, np.dtype(dtype).name).cpu().numpy()
    b = pw.apply_forward(x_true)
    oc = _core.SolverOptions(max_iters=6, ground_truth=x_true)
    ow = ctk.SolverOptions(max_iters=6, ground_truth=x_true)
    cases = [
        (lambda: _core.cgls(pc, b, oc), lambda: ctk.cgls(pw, b, ow)),
        (lambda: _core.lsqr(pc, b, oc), lambda: ctk.lsqr(pw, b, ow)),
        (lambda: _core.lsmr(pc, b, 0.5, oc), lambda: ctk.lsmr(pw, b, 0.5, ow)),
        (lambda: _core.hybrid_lsqr(pc, b, _core.HybridStrategy.gcv(), oc),
         lambda: ctk.hybrid_lsqr(pw, b, ctk.HybridStrategy.gcv(), ow)),
        (lambda: _core.cgls_tv(pc, b, 0.1, 2, 3, oc), lambda: ctk.cgls_tv(pw, b, 0.1, 2, 3, ow)),
        (lambda: _core.sirt(pc, b, oc), lambda: ctk.sirt(pw, b, ow)),
    ]
    for fc, fw in cases:
        rc, rw = fc(), fw()
        assert np.array_equal(rc.x, rw.x), rc.log.solver
        assert rc.iterations_run == rw.iterations_run and int(rc.stop_reason) == int(rw.stop_reason)
        assert rc.log.explicit_residual == rw.log.explicit_residual
        assert rc.log.implicit_residual == rw.log.implicit_residual
        assert rc.log.relative_error == rw.log.relative_error
        assert rc.log.lambda_ == rw.log.lambda_
        assert list(rc.outer_starts) == list(rw.outer_starts)
