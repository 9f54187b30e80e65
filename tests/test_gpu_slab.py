"""z-slab sharding on the device.

Kernel side, one process: a handle restricted to slices [z0, z0+n) is the operator of
the volume with x zero outside the slab, so (linearity) the slab forwards of a partition
sum to the full forward, and the slab backprojection is the full one restricted to the
slab -- bit-identical, since a voxel's contributions are summed in the same order.

Solver side: two processes on the one GPU, each owning one slab, with the product's
collectives over gloo (host-staged; no kernel waits on another rank), must reproduce the
unsharded solve for every solver (A x partials sum-reduced, domain dots and the domain-basis
CGS2 coefficients summed in rank order; CGLS-TV / flsqr_tv also the one-slice halos of the
gradient stencils)."""
import os
import socket
import sys

import numpy as np
import pytest

from geoms import cone_bench, to_ctk
from conftest import rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctk():
    import paper_2211_14212_b200 as m

    m.load()
    return m


def _slabs(nz, world):
    from paper_2211_14212_b200.comm import shard_slabs

    return [shard_slabs(nz, world, r) for r in range(world)]


@pytest.mark.parametrize("name", ["bench", "zrays"])
@pytest.mark.parametrize("variant", ["matched", "voxel_driven"])
def test_slab_operators_partition(ctk, name, variant):
    import torch

    if name == "bench":
        g = to_ctk(cone_bench(40, 24))
    else:  # short source distance: the outer detector rows are z-dominant rays
        g = ctk.ConeGeometry(ctk.BeamMode.cone3d, 40.0, 30.0, 1.5, 40, 128, ctk.VolumeShape(40, 40, 40, 1.0),
                             ctk.equidistant_angles(24))
    v = getattr(ctk.BackprojectVariant, variant)
    full = ctk.projector_pair(g, v)
    n = g.vol.nx * g.vol.ny
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.random(full.domain_size, dtype=np.float32)).cuda()
    y = torch.from_numpy(rng.random(full.range_size, dtype=np.float32)).cuda()
    ax_full = full.apply_forward(x)
    bt_full = full.apply_back(y)
    acc = torch.zeros_like(ax_full, dtype=torch.float64)
    for z0, cnt in _slabs(g.vol.nz, 3):
        p = ctk.projector_pair(g, v, slab=(z0, cnt))
        assert p.domain_size == n * cnt and p.domain_shape.nz == cnt
        acc += p.apply_forward(x[z0 * n:(z0 + cnt) * n].contiguous()).double()
        bt = p.apply_back(y)
        assert torch.equal(bt, bt_full[z0 * n:(z0 + cnt) * n]), "slab A^T b must be the restriction of the full one"
    assert rel_l2(acc.cpu().numpy(), ax_full.double().cpu().numpy()) < 2e-6


def test_slab_unsupported_paths(ctk):
    g = to_ctk(cone_bench(16, 8))
    p = ctk.projector_pair(g, dtype=np.float64, slab=(0, 8))
    with pytest.raises(ctk.UnsupportedError):
        p.apply_forward(np.zeros(p.domain_size))
    with pytest.raises(ctk.ParameterError):
        ctk.projector_pair(g, slab=(10, 8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    sys.path.insert(0, ROOT)
    from oracle.oracle import Restated, bench_geometry

    orc = Restated()
    g = bench_geometry(24, 16)
    gt = orc.shepp_logan_3d(24, np.float64)
    b = orc.forward(g, gt).astype(np.float32)
    return g, gt.astype(np.float32), b


SOLVERS = ["cgls", "lsqr", "lsmr", "sirt", "hybrid_lsqr", "ab_gmres", "ba_gmres", "cgls_tv", "flsqr_tv"]


def _solve(ctk, pair, b, which):
    opts = ctk.SolverOptions(max_iters=4 if which == "flsqr_tv" else 6, stop_on_explicit_residual_increase=False,
                             residual_tolerance=0.0)
    if which == "lsmr":
        return ctk.lsmr(pair, b, 5.0, opts)
    if which in ("hybrid_lsqr", "flsqr_tv"):
        return getattr(ctk, which)(pair, b, ctk.HybridStrategy.gcv(), opts)
    if which == "cgls_tv":
        return ctk.cgls_tv(pair, b, 0.5, 2, 3, opts)
    return getattr(ctk, which)(pair, b, opts)


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import paper_2211_14212_b200 as ctk
    from geoms import to_ctk as _to_ctk
    from paper_2211_14212_b200.comm import TorchComm, shard_slabs

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, gt, b = _problem()
    z0, cnt = shard_slabs(g.nz, world, rank)
    comm = TorchComm(rank, world, device="cuda")
    out = {}
    for which in SOLVERS:
        pair = ctk.projector_pair(_to_ctk(g), slab=(z0, cnt))
        pair.projector.attach_comm(comm)
        r = _solve(ctk, pair, b, which)
        out[which + "_x"] = r.x
        out[which + "_expl"] = np.array(r.log.explicit_residual)
        out[which + "_impl"] = np.array(r.log.implicit_residual)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), z0=z0, cnt=cnt, **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_slab_sharded_solvers_two_ranks(ctk, tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g, gt, b = _problem()
    n = g.nx * g.ny
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for which in SOLVERS:
        ref = _solve(ctk, ctk.projector_pair(to_ctk(g)), b, which)
        x = np.concatenate([r[which + "_x"] for r in ranks])
        assert x.size == n * g.nz
        assert rel_l2(x, ref.x) < 1e-4, which
        for r in ranks:  # every rank logs the same (global) residual history
            assert np.allclose(r[which + "_expl"], ref.log.explicit_residual, rtol=1e-4), which
            assert np.allclose(r[which + "_impl"], ref.log.implicit_residual, rtol=1e-4), which
        assert np.array_equal(ranks[0][which + "_expl"], ranks[1][which + "_expl"])


def _ops_worker(rank, world, port, outdir):
    """The public operators of a slab handle with a communicator attached (unequal slab
    heights): A x must be the reduced whole projection, A^T b the local restriction, and
    the fused residual the reduced one."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import paper_2211_14212_b200 as ctk
    from geoms import cone_bench as _cb, to_ctk as _to_ctk
    from paper_2211_14212_b200.comm import TorchComm, shard_slabs

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = _to_ctk(_cb(25, 12))
    n = g.vol.nx * g.vol.ny
    z0, cnt = shard_slabs(g.vol.nz, world, rank)
    rng = np.random.default_rng(11)
    x = rng.standard_normal(n * g.vol.nz).astype(np.float32)
    y = rng.standard_normal(g.nu * g.nv * len(g.angles)).astype(np.float32)
    comm = TorchComm(rank, world, device="cuda")
    p = ctk.projector_pair(g, slab=(z0, cnt))
    p.projector.attach_comm(comm)
    xs = torch.from_numpy(x[z0 * n:(z0 + cnt) * n].copy()).cuda()
    ax = p.apply_forward(xs).cpu().numpy()
    bt = p.apply_back(torch.from_numpy(y).cuda()).cpu().numpy()
    r2 = p.projector.residual2(xs, torch.from_numpy(y).cuda())
    np.savez(os.path.join(outdir, f"ops{rank}.npz"), z0=z0, cnt=cnt, ax=ax, bt=bt, r2=r2)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_slab_public_operators_with_comm_three_ranks(ctk, tmp_path):
    import torch.multiprocessing as mp

    world = 3
    mp.spawn(_ops_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = to_ctk(cone_bench(25, 12))
    n = g.vol.nx * g.vol.ny
    rng = np.random.default_rng(11)
    x = rng.standard_normal(n * g.vol.nz).astype(np.float32)
    y = rng.standard_normal(g.nu * g.nv * len(g.angles)).astype(np.float32)
    full = ctk.projector_pair(g)
    ax_full = full.apply_forward(x)
    bt_full = full.apply_back(y)
    r2_full = float(np.sum((ax_full.astype(np.float64) - y) ** 2))
    ranks = [np.load(tmp_path / f"ops{r}.npz") for r in range(world)]
    assert sorted(int(r["cnt"]) for r in ranks) == [8, 8, 9]
    for r in ranks:
        assert rel_l2(r["ax"], ax_full) < 2e-6  # the reduced whole projection on every rank
        z0, cnt = int(r["z0"]), int(r["cnt"])
        assert np.array_equal(r["bt"], bt_full[z0 * n:(z0 + cnt) * n])  # local, not summed
        assert abs(float(r["r2"]) - r2_full) <= 1e-5 * r2_full
    assert np.array_equal(ranks[0]["ax"], ranks[1]["ax"]) and np.array_equal(ranks[1]["ax"], ranks[2]["ax"])
