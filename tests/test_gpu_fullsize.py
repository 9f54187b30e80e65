"""Size-independent properties at BASELINE.json's full C3 size (512^3 volume, 512^2
detector, 360 views; the oracle cannot run there): adjointness of the matched f32 pair,
linearity, the slab partition, A^T b restriction, and bitwise rerun determinism of a solve.
Also the C2 Siddon pair at its full size (256^3, 180 views)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctk():
    import paper_2211_14212_b200 as m

    m.load()
    return m


@pytest.fixture(scope="module")
def c3(ctk):
    import torch

    g = ctk.bench_geometry(512, 360)
    pair = ctk.projector_pair(g)
    gen = torch.Generator(device="cuda").manual_seed(11)
    x = torch.rand(pair.domain_size, device="cuda", generator=gen)
    y = torch.rand(pair.range_size, device="cuda", generator=gen)
    return g, pair, x, y


def _dot(a, b):
    return float((a.double() * b.double()).sum())


def test_c3_matched_adjoint(ctk, c3):
    g, pair, x, y = c3
    ax = pair.apply_forward(x)
    aty = pair.apply_back(y)
    lhs, rhs = _dot(ax, y), _dot(x, aty)
    assert abs(lhs - rhs) <= 2e-6 * abs(lhs)  # same f32 positions and weights both ways


def test_c3_linearity_and_determinism(ctk, c3):
    import torch

    g, pair, x, y = c3
    x2 = torch.flip(x, [0]).contiguous()
    a1, a2 = pair.apply_forward(x), pair.apply_forward(x2)
    a12 = pair.apply_forward(x + x2)
    rel = float((a12.double() - a1.double() - a2.double()).norm() / a12.double().norm())
    assert rel < 1e-6
    assert torch.equal(pair.apply_forward(x), a1)  # bitwise rerun
    b1 = pair.apply_back(y)
    assert torch.equal(pair.apply_back(y), b1)


def test_c3_slab_partition(ctk, c3):
    import torch

    from paper_2211_14212_b200.comm import shard_slabs

    g, pair, x, y = c3
    n = 512 * 512
    full_ax = pair.apply_forward(x)
    full_bt = pair.apply_back(y)
    acc = torch.zeros_like(full_ax, dtype=torch.float64)
    for r in range(4):
        z0, cnt = shard_slabs(512, 4, r)
        p = ctk.projector_pair(g, slab=(z0, cnt))
        acc += p.apply_forward(x[z0 * n:(z0 + cnt) * n].contiguous()).double()
        assert torch.equal(p.apply_back(y), full_bt[z0 * n:(z0 + cnt) * n])
    assert float((acc - full_ax.double()).norm() / full_ax.double().norm()) < 2e-6


def test_c3_lsmr_rerun_bitwise(ctk, c3):
    g, pair, x, y = c3
    b = pair.apply_forward(ctk.shepp_logan_3d(512))
    opts = ctk.SolverOptions(max_iters=3, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)
    r1 = ctk.lsmr(pair, b, 30.0, opts)
    r2 = ctk.lsmr(pair, b, 30.0, opts)
    assert r1.log.explicit_residual == r2.log.explicit_residual
    assert r1.log.implicit_residual == r2.log.implicit_residual
    expl = r1.log.explicit_residual
    assert expl[0] > expl[1] > expl[2]  # LSMR's residual decreases on consistent data


def test_c2_siddon_adjoint(ctk):
    import torch

    g = ctk.bench_geometry(256, 180)
    pair = ctk.projector_pair(g, projector=ctk.ProjectorKind.siddon)
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(pair.domain_size, device="cuda", generator=gen)
    y = torch.rand(pair.range_size, device="cuda", generator=gen)
    lhs, rhs = _dot(pair.apply_forward(x), y), _dot(x, pair.apply_back(y))
    assert abs(lhs - rhs) <= 2e-6 * abs(lhs)


def test_wide_offset_instantiation_matches(tmp_path):
    """The 64-bit-offset forward (volumes beyond ~1290^3) forced on a small problem must give
    the same projections as the 32-bit one."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np, torch; sys.path.insert(0, %r); import paper_2211_14212_b200 as ctk; "
            "g = ctk.bench_geometry(64, 30); p = ctk.projector_pair(g); x = ctk.shepp_logan_3d(64); "
            "y = p.apply_forward(x); np.save(sys.argv[1], y.cpu().numpy())") % root
    outs = []
    for wide in ("0", "1"):
        f = str(tmp_path / f"y{wide}.npy")
        subprocess.run([sys.executable, "-c", code, f], check=True, env={**os.environ, "CTK_FWD_WIDE": wide})
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def _subset_geom(n, na_total, views):
    from oracle.oracle import CONE3D, Geom, equidistant_angles

    ang = np.array(equidistant_angles(na_total))[np.linspace(0, na_total - 1, views).astype(int)]
    return Geom(CONE3D, 2.0 * n, 1.0 * n, 1.5, n, n, n, n, n, 1.0, ang)


def _rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("views", [4, 16])
def test_c3_parity_on_view_subset(ctk, reference, views):
    """The north-star bar at the full C3 size: the reference T=double Ax and matched A^T b
    (oracle/_ref, the box's host threads) on 4 / 16 of the 360 views of the 512^3 / 512^2
    acquisition, on the Shepp-Logan phantom and its projections AND on random-signed data
    (the operand LSQR/LSMR actually pass to A^T b); f32 within half the 1e-5 bar."""
    import os

    import torch

    from geoms import to_ctk

    n = 512
    g = _subset_geom(n, 360, views)
    reference.set_threads(min(16, os.cpu_count() or 1))
    try:
        p = ctk.projector_pair(to_ctk(g))
        x = ctk.make_phantom(ctk.PhantomKind.shepp_logan_3d, n, "float64").cpu().numpy()
        yr = reference.forward(g, x)
        br = reference.back(g, yr, 0)
        assert _rel(p.apply_forward(x.astype(np.float32)), yr) < 5e-6    # measured 1.7e-7
        assert _rel(p.apply_back(yr.astype(np.float32)), br) < 5e-6      # measured 0.9-1.4e-7
        rng = np.random.default_rng(3)
        xs = rng.standard_normal(g.domain_size, dtype=np.float32).astype(np.float64)
        ys = rng.standard_normal(g.range_size, dtype=np.float32).astype(np.float64)
        assert _rel(p.apply_forward(torch.from_numpy(xs.astype(np.float32)).cuda()), reference.forward(g, xs)) < 5e-6
        assert _rel(p.apply_back(torch.from_numpy(ys.astype(np.float32)).cuda()), reference.back(g, ys, 0)) < 5e-6
    finally:
        reference.set_threads(1)


@pytest.mark.timeout(1500)
def test_c5_parity_on_view_subset_signed(ctk, reference):
    """C5 extents (1024^3 volume, 1024^2 detector) on 4 of the 1600 views, random-signed
    data: f32 Ax and matched A^T b within half the 1e-5 bar of the reference T=double.
    (4 reference threads: its matched scatter keeps one 8 GiB partial volume per thread.)"""
    import torch

    from geoms import to_ctk

    n = 1024
    g = _subset_geom(n, 1600, 4)
    reference.set_threads(4)
    try:
        p = ctk.projector_pair(to_ctk(g))
        rng = np.random.default_rng(7)
        xs = rng.standard_normal(g.domain_size, dtype=np.float32)
        ax = p.apply_forward(torch.from_numpy(xs).cuda()).cpu().numpy()
        yref = reference.forward(g, xs.astype(np.float64))
        assert _rel(ax, yref) < 5e-6
        del xs, ax, yref
        ys = rng.standard_normal(g.range_size, dtype=np.float32)
        bt = p.apply_back(torch.from_numpy(ys).cuda()).cpu().numpy()
        bref = reference.back(g, ys.astype(np.float64), 0)
        assert _rel(bt, bref) < 5e-6
    finally:
        reference.set_threads(1)
