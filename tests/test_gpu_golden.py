"""The product against the committed golden fixtures (tests/golden/*.npz, generated from the
reference by tests/golden/make_golden.py), so GPU parity does not depend on oracle/_ref being
present: f64 operators bit-exact, f32 within 1e-5, the f64 device solvers (5 iterations of
CGLS / LSQR / LSMR lambda=3) within 1e-9 of the reference's T=double solves."""
import glob
import os

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _geom(ctk, d):
    return ctk.ConeGeometry(ctk.BeamMode(int(d["mode"])), float(d["dso"]), float(d["dod"]), float(d["du"]),
                            int(d["nu"]), int(d["nv"]),
                            ctk.VolumeShape(int(d["nx"]), int(d["ny"]), int(d["nz"]), float(d["h"])),
                            list(np.asarray(d["angles"], dtype=np.float64)))


def test_golden_fixtures_present():
    assert len(GOLDEN) >= 4, "tests/golden/*.npz missing"


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_operators_match_golden(path):
    import paper_2211_14212_b200 as ctk

    d = np.load(path)
    g = _geom(ctk, d)
    p64 = ctk.projector_pair(g, dtype=np.float64)
    assert np.array_equal(p64.apply_forward(d["x"]), d["ax"])
    assert np.array_equal(p64.apply_back(d["y"]), d["atb_matched"])
    pv = ctk.projector_pair(g, ctk.BackprojectVariant.voxel_driven, dtype=np.float64)
    assert np.array_equal(pv.apply_back(d["y"]), d["atb_voxel"])
    p32 = ctk.projector_pair(g)
    assert rel_l2(p32.apply_forward(d["x"].astype(np.float32)), d["ax"]) < 1e-5
    assert rel_l2(p32.apply_back(d["y"].astype(np.float32)), d["atb_matched"]) < 1e-5


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_solvers_match_golden(path):
    import paper_2211_14212_b200 as ctk

    d = np.load(path)
    pair = ctk.projector_pair(_geom(ctk, d), dtype=np.float64)
    o = ctk.SolverOptions(max_iters=5, residual_tolerance=0.0, stop_on_explicit_residual_increase=False)
    for name, res in (("cgls", ctk.cgls(pair, d["b"], o)), ("lsqr", ctk.lsqr(pair, d["b"], o)),
                      ("lsmr", ctk.lsmr(pair, d["b"], 3.0, o))):
        assert rel_l2(res.x, d[f"{name}_x"]) < 1e-9, name
        assert np.allclose(res.log.explicit_residual, d[f"{name}_explicit"], rtol=1e-9), name
        assert np.allclose(res.log.implicit_residual, d[f"{name}_implicit"], rtol=1e-9), name
