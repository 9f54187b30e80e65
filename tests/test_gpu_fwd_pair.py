"""The two-volume forward march (ax2_f32, fwd_f32.cu) inside the solvers.

lsqr, lsmr and hybrid_lsqr announce their next A v before the monitor records an iterate
(cgls and cgls_tv advance their recurrence first to have the next A p); the explicit
residual's A x (solve_log.hpp:102-115) and that product then run as one march over
interleaved layouts.  Each output is bit-identical to a single-volume launch, so every
solve must be bitwise the same with the pairing switched off (CTK_FWD_NO_PAIR=1): x, both
residual histories, lambda and relative-error logs.  The geometries cover x- and
y-dominant rays, z-dominant rays (cone_steep), odd slice counts and ragged extents.
"""
import os

import numpy as np
import pytest

from geoms import ALL, cone_bench, to_ctk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctk():
    import paper_2211_14212_b200 as m

    m.load()
    return m


def _solve(ctk, pair, b, solver, k, paired, tol=0.0):
    if paired:
        os.environ.pop("CTK_FWD_NO_PAIR", None)
    else:
        os.environ["CTK_FWD_NO_PAIR"] = "1"
    try:
        opts = ctk.SolverOptions(max_iters=k, stop_on_explicit_residual_increase=False, residual_tolerance=tol)
        if solver == "lsmr":
            return ctk.lsmr(pair, b, 3.0, opts)
        if solver == "hybrid_lsqr":
            return ctk.hybrid_lsqr(pair, b, ctk.HybridStrategy.gcv(), opts)
        if solver == "cgls":
            return ctk.cgls(pair, b, opts)
        if solver == "cgls_tv":
            return ctk.cgls_tv(pair, b, 0.05, 2, 4, opts, warm_start=True)
        return ctk.lsqr(pair, b, opts)
    finally:
        os.environ.pop("CTK_FWD_NO_PAIR", None)


def _same(r1, r2):
    assert r1.iterations_run == r2.iterations_run
    assert r1.stop_reason == r2.stop_reason
    assert np.array_equal(r1.x, r2.x)
    assert r1.log.implicit_residual == r2.log.implicit_residual
    assert r1.log.explicit_residual == r2.log.explicit_residual
    assert r1.log.lambda_ == r2.log.lambda_


@pytest.mark.parametrize("solver", ["lsqr", "lsmr", "hybrid_lsqr", "cgls", "cgls_tv"])
@pytest.mark.parametrize("name", ["cone_default", "cone_steep", "cone_ragged", "parallel3d", "cone_multitile"])
def test_paired_residual_bitwise(ctk, name, solver):
    g = ALL[name]()
    rng = np.random.default_rng(7)
    b = rng.standard_normal(g.na * g.nv * g.nu).astype(np.float32)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32)
    k = 8 if solver == "cgls_tv" else 6
    _same(_solve(ctk, pair, b, solver, k, True), _solve(ctk, pair, b, solver, k, False))


@pytest.mark.parametrize("name", ["cone_default", "cone_steep", "cone_ragged", "parallel3d"])
def test_paired_residual_bitwise_siddon(ctk, name):
    # the f32 Siddon slab model (k_ax2_zfast_f32<SID=1>) and its z-ray DDA
    g = ALL[name]()
    b = np.random.default_rng(9).standard_normal(g.na * g.nv * g.nu).astype(np.float32)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32, projector=ctk.ProjectorKind.siddon)
    _same(_solve(ctk, pair, b, "lsqr", 6, True), _solve(ctk, pair, b, "lsqr", 6, False))


@pytest.mark.parametrize("solver", ["cgls", "lsqr", "cgls_tv"])
def test_paired_tolerance_stop(ctk, solver):
    # a tolerance stop mid-run: the advanced recurrence (cgls) and the announced product go
    # unused, the solve ends at the same iteration with the same x
    g = ALL["cone_default"]()
    b = np.abs(np.random.default_rng(4).standard_normal(g.na * g.nv * g.nu)).astype(np.float32)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32)
    full = _solve(ctk, pair, b, solver, 8, False)
    tol = full.log.explicit_residual[2] * (1 + 1e-9)
    r1, r2 = _solve(ctk, pair, b, solver, 8, True, tol), _solve(ctk, pair, b, solver, 8, False, tol)
    assert r1.iterations_run <= 3 < 8
    _same(r1, r2)


@pytest.mark.parametrize("solver", ["cgls_tv", "lsqr"])
def test_paired_residual_whole_slab(ctk, solver):
    # a z-slab handle holding every slice (bench --shard slab at one rank) pairs too
    g = ALL["cone_ragged"]()
    b = np.random.default_rng(6).standard_normal(g.na * g.nv * g.nu).astype(np.float32)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32, slab=(0, g.nz))
    k = 8 if solver == "cgls_tv" else 6
    _same(_solve(ctk, pair, b, solver, k, True), _solve(ctk, pair, b, solver, k, False))


def test_paired_residual_bench_geometry(ctk):
    # 128^3 with several slice chunks per ray (fwd_chunks) and 90 views
    g = cone_bench(128, 90)
    rng = np.random.default_rng(11)
    b = np.abs(rng.standard_normal(g.na * g.nv * g.nu)).astype(np.float32)
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32)
    _same(_solve(ctk, pair, b, "lsmr", 4, True), _solve(ctk, pair, b, "lsmr", 4, False))


def test_paired_residual_wide_offsets(tmp_path):
    # the 64-bit-offset instantiation (CTK_FWD_WIDE=1 is read once per process)
    import subprocess
    import sys

    code = r'''
import os, sys
import numpy as np
sys.path.insert(0, "tests")
import paper_2211_14212_b200 as ctk
from geoms import cone_ragged, to_ctk
ctk.load()
g = cone_ragged()
b = np.random.default_rng(3).standard_normal(g.na * g.nv * g.nu).astype(np.float32)
pair = ctk.projector_pair(to_ctk(g), dtype=np.float32)
def run():
    opts = ctk.SolverOptions(max_iters=5, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)
    return ctk.lsqr(pair, b, opts)
r1 = run()
os.environ["CTK_FWD_NO_PAIR"] = "1"
r2 = run()
assert np.array_equal(r1.x, r2.x)
assert r1.log.explicit_residual == r2.log.explicit_residual
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {**os.environ, "CTK_FWD_WIDE": "1"}
    env.pop("CTK_FWD_NO_PAIR", None)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("projector", ["joseph", "siddon"])
@pytest.mark.parametrize("name", ["cone_default", "cone_steep", "parallel3d", "cone_multitile"])
def test_forward_pair_bitwise(ctk, name, projector):
    import torch

    g = ALL[name]()
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32, projector=ctk.ProjectorKind[projector])
    gen = torch.Generator(device="cuda").manual_seed(5)
    x1 = torch.randn(g.nx * g.ny * g.nz, device="cuda", generator=gen)
    x2 = torch.randn(g.nx * g.ny * g.nz, device="cuda", generator=gen)
    y1, y2 = (torch.full((pair.range_size,), float("nan"), device="cuda") for _ in range(2))
    z1, z2 = (torch.empty(pair.range_size, device="cuda") for _ in range(2))
    pair.projector.forward_pair(x1, y1, x2, y2)
    pair.forward(x1, z1)
    pair.forward(x2, z2)
    torch.cuda.synchronize()
    assert torch.equal(y1, z1) and torch.equal(y2, z2)


def test_forward_pair_unsupported(ctk):
    import torch

    g = ALL["cone_default"]()
    pair = ctk.projector_pair(to_ctk(g), dtype=np.float32, slab=(4, 8))  # a z-slab handle
    x = torch.zeros(pair.domain_size, device="cuda")
    y = torch.zeros(pair.range_size, device="cuda")
    with pytest.raises(ctk.UnsupportedError):
        pair.projector.forward_pair(x, y, x, y)
