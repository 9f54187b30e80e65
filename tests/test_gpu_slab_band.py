"""Band-sharded range of z-slab sharding (bands.cpp) through the product
operators and solvers: three processes on the one GPU, collectives over gloo (host-staged,
no kernel waits on another rank; the exchanges are point-to-point sends/receives).

Each rank holds its slab of the volume AND only its detector-row window of every range
vector (the rows its slab's rays reach plus the rows it owns, non-owned rows zero):
 * A x: the owned rows equal the whole projection's rows (partials summed by the owner in
   rank order), the other held rows are zero;
 * A^T b: bit-identical to the whole back projection restricted to the slab (the halo rows
   come from their owners);
 * every solver reproduces the unsharded solve, with identical logs on every rank."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import rel_l2
from geoms import cone_bench, to_ctk

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _geom(name="cone"):
    if name == "parallel3d":
        from geoms import parallel3d

        return to_ctk(parallel3d(nx=20, ny=18, nz=30, na=12))
    return to_ctk(cone_bench(36, 20))


def _ops_worker(rank, world, port, outdir, name="cone"):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200.comm import TorchComm, shard_slabs

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = _geom(name)
    n = g.vol.nx * g.vol.ny
    z0, cnt = shard_slabs(g.vol.nz, world, rank)
    rng = np.random.default_rng(7)
    x = rng.standard_normal(n * g.vol.nz).astype(np.float32)
    y = rng.standard_normal(g.nu * g.nv * len(g.angles)).astype(np.float32)
    comm = TorchComm(rank, world, device="cuda")
    p = ctk.projector_pair(g, slab=(z0, cnt), comm=comm, shard_range=True)
    w0, nw, o0, no = p.projector.range_rows()
    ax = p.apply_forward(torch.from_numpy(x[z0 * n:(z0 + cnt) * n].copy()).cuda()).cpu().numpy()
    yl = p.projector.local_range(y)
    bt = p.apply_back(torch.from_numpy(yl).cuda()).cpu().numpy()
    np.savez(os.path.join(outdir, f"ops{rank}.npz"), z0=z0, cnt=cnt, w0=w0, nw=nw, o0=o0, no=no, ax=ax, bt=bt,
             rs=p.range_size)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("name", ["cone", "parallel3d"])
def test_band_operators_three_ranks(tmp_path, name):
    import torch.multiprocessing as mp

    import paper_2211_14212_b200 as ctk

    mp.spawn(_ops_worker, args=(WORLD, _free_port(), str(tmp_path), name), nprocs=WORLD, join=True)
    g = _geom(name)
    n, na = g.vol.nx * g.vol.ny, len(g.angles)
    rng = np.random.default_rng(7)
    x = rng.standard_normal(n * g.vol.nz).astype(np.float32)
    y = rng.standard_normal(g.nu * g.nv * na).astype(np.float32)
    full = ctk.projector_pair(g)
    ax_full = full.apply_forward(x).reshape(na, g.nv, g.nu)
    bt_full = full.apply_back(y)
    ranks = [np.load(tmp_path / f"ops{r}.npz") for r in range(WORLD)]
    owned = []
    for r in ranks:
        w0, nw, o0, no = (int(r[k]) for k in ("w0", "nw", "o0", "no"))
        assert int(r["rs"]) == na * nw * g.nu and (nw < g.nv or name != "cone")  # a window, not the whole range
        ax = r["ax"].reshape(na, nw, g.nu)
        own = ax[:, o0 - w0:o0 - w0 + no, :]
        assert rel_l2(own, ax_full[:, o0:o0 + no, :]) < 2e-6
        assert not np.any(ax[:, :o0 - w0, :]) and not np.any(ax[:, o0 - w0 + no:, :])  # held, not owned: 0
        owned.append((o0, no))
        z0, cnt = int(r["z0"]), int(r["cnt"])
        assert np.array_equal(r["bt"], bt_full[z0 * n:(z0 + cnt) * n])
    assert owned[0][0] == 0 and sum(no for _, no in owned) == g.nv


SOLVERS = ["cgls", "lsqr", "lsmr", "sirt", "hybrid_lsqr", "ab_gmres", "ba_gmres", "cgls_tv", "flsqr_tv"]


def _problem():
    sys.path.insert(0, ROOT)
    from oracle.oracle import Restated, bench_geometry

    orc = Restated()
    g = bench_geometry(36, 20)
    gt = orc.shepp_logan_3d(36, np.float64)
    b = orc.forward(g, gt).astype(np.float32)
    return g, b


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


def _solve_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import paper_2211_14212_b200 as ctk
    from geoms import to_ctk as _to_ctk
    from paper_2211_14212_b200.comm import TorchComm, shard_slabs

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, b = _problem()
    z0, cnt = shard_slabs(g.nz, world, rank)
    comm = TorchComm(rank, world, device="cuda")
    out = {}
    for which in SOLVERS:
        pair = ctk.projector_pair(_to_ctk(g), slab=(z0, cnt), comm=comm, shard_range=True)
        bl = pair.projector.local_range(b)
        r = _solve(ctk, pair, bl, which)
        out[which + "_x"] = r.x
        out[which + "_expl"] = np.array(r.log.explicit_residual)
        out[which + "_impl"] = np.array(r.log.implicit_residual)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_band_sharded_solvers_three_ranks(tmp_path):
    import torch.multiprocessing as mp

    import paper_2211_14212_b200 as ctk

    mp.spawn(_solve_worker, args=(WORLD, _free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    g, b = _problem()
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(WORLD)]
    for which in SOLVERS:
        ref = _solve(ctk, ctk.projector_pair(to_ctk(g)), b, which)
        x = np.concatenate([r[which + "_x"] for r in ranks])
        assert rel_l2(x, ref.x) < 1e-4, which
        for r in ranks:
            assert np.allclose(r[which + "_expl"], ref.log.explicit_residual, rtol=1e-4), which
            assert np.allclose(r[which + "_impl"], ref.log.implicit_residual, rtol=1e-4), which
        assert np.array_equal(ranks[0][which + "_expl"], ranks[2][which + "_expl"]), which


def test_band_needs_slab_and_comm():
    import paper_2211_14212_b200 as ctk

    g = _geom()
    p = ctk.projector_pair(g, slab=(0, 12))
    with pytest.raises(ctk.ParameterError, match="needs a slab and a communicator"):
        p.projector.shard_range()
