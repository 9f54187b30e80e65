"""GPU Siddon exact-length projector (new code).

No reference implementation exists, so the checker is the C restatement
(oracle/ctk_oracle.c), itself pinned by the reference's ray-box chord KAT
(tests/test_oracle.py::test_siddon_*).  f64 is held BIT-EXACT to the restatement; f32 (the
slab-model kernels that share the Joseph layouts) within 5e-6 of it on signed data; the
transposes pass the adjoint test; LSQR on the Siddon pair matches the
numpy solver restatement (pinned against the reference solvers) at config-2 shape."""
import math

import numpy as np
import pytest

from geoms import ALL, cone_bench, to_ctk
from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctk():
    import paper_2211_14212_b200 as m

    m.load()
    return m


def _pair(ctk, g, dtype):
    return ctk.projector_pair(to_ctk(g), dtype=dtype, projector=ctk.ProjectorKind.siddon)


@pytest.mark.parametrize("name", sorted(ALL))
@pytest.mark.parametrize("dtype", [np.float64])
def test_siddon_bit_exact_vs_restatement(ctk, restated, name, dtype):
    g = ALL[name]()
    rng = np.random.default_rng(3)
    x = rng.standard_normal(g.domain_size).astype(dtype)
    y = rng.standard_normal(g.range_size).astype(dtype)
    y[::6] = 0
    pair = _pair(ctk, g, dtype)
    assert np.array_equal(pair.apply_forward(x), restated.siddon_forward(g, x))
    assert np.array_equal(pair.apply_back(y), restated.siddon_back(g, y))


@pytest.mark.parametrize("name", sorted(ALL))
def test_siddon_f32_slab_model_within_1e5(ctk, restated, name):
    """The f32 Siddon pair (slab decomposition along the dominant axis with anchored f32
    cell positions, f32_common.cuh; z-dominant rays by the exact DDA / gather) against the
    f64 restatement, random-signed data (the cancelling inputs LSQR feeds A^T b)."""
    g = ALL[name]()
    rng = np.random.default_rng(11)
    x = rng.standard_normal(g.domain_size)
    y = rng.standard_normal(g.range_size)
    pair = _pair(ctk, g, np.float32)
    ef = rel_l2(pair.apply_forward(x.astype(np.float32)), restated.siddon_forward(g, x))
    eb = rel_l2(pair.apply_back(y.astype(np.float32)), restated.siddon_back(g, y))
    assert ef < 5e-6 and eb < 5e-6, (ef, eb)


def test_siddon_f32_within_1e5_of_f64(ctk, restated):
    g = cone_bench(32, 20)
    x = restated.shepp_logan_3d(32, np.float64)
    want = restated.siddon_forward(g, x)
    got = _pair(ctk, g, np.float32).apply_forward(x.astype(np.float32))
    assert rel_l2(got, want) < 1e-5


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-10), (np.float32, 2e-6)])
def test_siddon_adjoint(ctk, dtype, tol):
    from oracle.oracle import adjoint_discrepancy

    for name in ("parallel2d", "cone_adjoint", "cone_ragged"):
        g = ALL[name]()
        pair = _pair(ctk, g, dtype)
        assert adjoint_discrepancy(pair.apply_forward, pair.apply_back, g.domain_size, g.range_size, 10, 5, dtype) < tol


def test_siddon_chord_kat(ctk):
    from oracle.oracle import ray_box_chord

    h, th, n = 0.9, 0.3, 7
    g = ctk.ConeGeometry(ctk.BeamMode.cone3d, 4.0 * n * h, 2.0 * n * h, h, 1, 1, ctk.VolumeShape(n, n, n, h), [th])
    x = np.zeros(n ** 3)
    x[n // 2 + n * (n // 2 + n * (n // 2))] = 1
    o = [g.source_to_origin * math.cos(th), g.source_to_origin * math.sin(th), 0.0]
    nn = math.hypot(o[0], o[1])
    chord = ray_box_chord(o, [-o[0] / nn, -o[1] / nn, 0.0], [-h / 2] * 3, [h / 2] * 3)
    y = ctk.projector_pair(g, dtype=np.float64, projector=ctk.ProjectorKind.siddon).apply_forward(x)
    assert y[0] == pytest.approx(chord, rel=1e-12)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_siddon_lsqr_config2_shape(ctk, restated, dtype):
    """Config 2's solver on the Siddon pair (LSQR), scaled to 32^3 / 32^2 / 24 views."""
    from oracle.oracle import lsqr

    g = cone_bench(32, 24)
    gt = restated.shepp_logan_3d(32, np.float64)
    b = restated.siddon_forward(g, gt)
    k = 8
    want = lsqr(lambda v: restated.siddon_forward(g, v), lambda v: restated.siddon_back(g, v), b, k, tol=0.0,
                stop_inc=False)
    res = ctk.lsqr(_pair(ctk, g, dtype), b.astype(dtype),
                   ctk.SolverOptions(max_iters=k, residual_tolerance=0.0, stop_on_explicit_residual_increase=False))
    assert rel_l2(res.x, want["x"]) < 1e-4
    assert np.allclose(res.log.explicit_residual, want["explicit"], rtol=1e-4)
    assert np.allclose(res.log.implicit_residual, want["implicit"], rtol=1e-4)
