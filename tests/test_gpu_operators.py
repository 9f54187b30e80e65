"""The reference's operator compositions and stencils on the device: gradient / its adjoint
and the IRN TV weights against the reference's gradient.hpp / tv.hpp (compiled unmodified,
oracle/_ref) -- bit-identical in double (TV weights: within an ulp, the device pow) -- and augment_tikhonov / stack_weighted_gradient
(operators.hpp:118-186): shapes, the adjoint identity, and agreement with the same
composition built from the reference's own projector."""
import ctypes as C

import numpy as np
import pytest

from conftest import rel_l2
from geoms import cone_adjoint, to_ctk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctk():
    import paper_2211_14212_b200 as m

    m.load()
    return m


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@pytest.mark.parametrize("shape", [(7, 5, 4), (16, 1, 1), (1, 9, 3), (12, 12, 12)])
def test_gradient_and_adjoint_bit_exact(ctk, reference, shape):
    nx, ny, nz = shape
    vs = ctk.VolumeShape(nx, ny, nz, 1.0)
    rng = np.random.default_rng(nx * 100 + ny * 10 + nz)
    x = rng.standard_normal(nx * ny * nz)
    want = [np.zeros_like(x) for _ in range(3)]
    assert reference.lib.ref_gradient_f64(nx, ny, nz, _fp(x), *[_fp(w) for w in want]) == 0
    got = ctk.gradient(x, vs)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    g3 = [rng.standard_normal(x.size) for _ in range(3)]
    adj = np.zeros_like(x)
    assert reference.lib.ref_gradient_adjoint_f64(nx, ny, nz, *[_fp(v) for v in g3], _fp(adj)) == 0
    assert np.array_equal(ctk.gradient_adjoint(*g3, vs), adj)


def test_tv_weights_match(ctk, reference):
    nx, ny, nz = 9, 8, 7
    x = np.random.default_rng(3).standard_normal(nx * ny * nz)
    want = np.zeros_like(x)
    assert reference.lib.ref_tv_weights_f64(nx, ny, nz, _fp(x), _fp(want)) == 0
    got = ctk.tv_weights(x, ctk.VolumeShape(nx, ny, nz, 1.0))
    # same fp64 operation sequence; only pow(m2 + eps^2, -1/4) comes from the CUDA libm
    # instead of glibc (within an ulp)
    assert np.max(np.abs(got - want) / want) <= 4.5e-16
    assert np.array_equal(ctk.tv_weights(np.zeros(8), ctk.VolumeShape(2, 2, 2, 1.0)), np.ones(8))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_compositions_adjoint_and_values(ctk, reference, dtype):
    g = cone_adjoint()
    pair = ctk.projector_pair(to_ctk(g), dtype=dtype)
    rng = np.random.default_rng(9)
    w = rng.random(pair.domain_size) + 0.5
    for op, extra in ((ctk.augment_tikhonov(pair, 0.7), pair.domain_size),
                      (ctk.stack_weighted_gradient(pair, 0.3, w), 3 * pair.domain_size)):
        assert op.range_size == pair.range_size + extra and op.domain_size == pair.domain_size
        x = rng.standard_normal(op.domain_size).astype(dtype)
        y = rng.standard_normal(op.range_size).astype(dtype)
        ax, aty = op.apply_forward(x), op.apply_back(y)
        lhs, rhs = float(np.dot(ax.astype(np.float64), y)), float(np.dot(x.astype(np.float64), aty))
        assert abs(lhs - rhs) <= (1e-10 if dtype == np.float64 else 2e-5) * abs(lhs)
        # the first block is the projector itself
        assert rel_l2(ax[:pair.range_size], reference.forward(g, x.astype(np.float64))) < (1e-12 if dtype == np.float64 else 1e-5)
    # explicit blocks in double
    if dtype == np.float64:
        op = ctk.augment_tikhonov(pair, 0.7)
        x = rng.standard_normal(op.domain_size)
        assert np.array_equal(op.apply_forward(x)[pair.range_size:], 0.7 * x)
        sg = ctk.stack_weighted_gradient(pair, 0.3, w)
        dx, dy, dz = ctk.gradient(x, pair.domain_shape)
        s = 0.3 * w
        assert np.array_equal(sg.apply_forward(x)[pair.range_size:], np.concatenate([s * dx, s * dy, s * dz]))
    with pytest.raises(ctk.ParameterError):
        ctk.augment_tikhonov(pair, -1.0)
    with pytest.raises(ctk.DimensionError):
        ctk.stack_weighted_gradient(pair, 0.3, w[:-1])
