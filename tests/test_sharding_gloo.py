"""Multi-rank host logic of angle sharding on CPU (gloo, world_size 2).

The product's sharding contract (solvers.cpp header): rank r owns the
contiguous angle block ctk_shard_angles(na, G, r); Ax is local; every A^T b partial volume
is sum-reduced; range-space reductions are all-gathered and summed in RANK ORDER.  Here the
per-rank operators are the CPU oracle (no GPU in this container) while the partition and
the collectives are the product's own (ctk_shard_angles, comm.TorchComm over gloo).  The
sharded LSQR recurrence must reproduce the unsharded one, and every rank must hold
bitwise-identical scalars and iterates."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C

    import torch
    import torch.distributed as dist

    from oracle.oracle import Restated, bench_geometry
    from paper_2211_14212_b200.comm import TorchComm, shard_angles

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    orc = Restated()
    g = bench_geometry(12, 10)
    gt = orc.shepp_logan_3d(12, np.float64)
    b_full = orc.forward(g, gt)
    first, count = shard_angles(g.na, world, rank)
    gs = g.subset(np.arange(first, first + count))
    frame = g.nu * g.nv
    b = b_full[first * frame:(first + count) * frame].copy()
    comm = TorchComm(rank, world, device="cpu")

    def atb(y):
        v = orc.back(gs, y)
        comm.allreduce_buffer(v.ctypes.data, v.size, 1)  # in place, f64
        return v

    def rnorm(y):
        return np.sqrt(comm.sum_scalar(float(y @ y)))

    # LSQR (solvers.hpp:62-126) with the sharded reductions of solvers.cpp
    k_max = 6
    beta1 = rnorm(b)
    u = b / beta1
    v = atb(u)
    alpha = float(np.linalg.norm(v))
    v = v / alpha
    w = v.copy()
    x = np.zeros_like(v)
    phibar, rhobar = beta1, alpha
    hist = []
    for _ in range(k_max):
        un = orc.forward(gs, v) - alpha * u
        beta = rnorm(un)
        u = un / beta
        vn = atb(u) - beta * v
        alpha = float(np.linalg.norm(vn))
        v = vn / alpha
        rho = np.hypot(rhobar, beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        x = x + (phi / rho) * w
        w = v - (theta / rho) * w
        expl = rnorm(orc.forward(gs, x) - b) / beta1
        hist.append((phibar / beta1, expl))
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), x=x, hist=np.array(hist), beta1=beta1)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_angle_sharded_lsqr_gloo(tmp_path):
    import torch.multiprocessing as mp

    from oracle.oracle import Restated, bench_geometry, lsqr

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    # every rank holds bitwise the same replicated state
    assert np.array_equal(r0["x"], r1["x"])
    assert np.array_equal(r0["hist"], r1["hist"])
    # and it reproduces the unsharded solve
    orc = Restated()
    g = bench_geometry(12, 10)
    gt = orc.shepp_logan_3d(12, np.float64)
    b = orc.forward(g, gt)
    want = lsqr(lambda v: orc.forward(g, v), lambda v: orc.back(g, v), b, 6, tol=0.0, stop_inc=False)
    assert np.linalg.norm(r0["x"] - want["x"]) <= 1e-10 * np.linalg.norm(want["x"])
    assert np.allclose(r0["hist"][:, 1], want["explicit"], rtol=1e-10)
    assert np.allclose(r0["hist"][:, 0], want["implicit"], rtol=1e-10)


def _sum_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2211_14212_b200.comm import TorchComm

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = TorchComm(rank, world, device="cpu")
    vals = [0.1 * (rank + 1), 1e16 if rank == 0 else 1.0, -1e16 if rank == 1 else 3.0]
    out = [comm.sum_scalar(v) for v in vals]
    np.save(os.path.join(outdir, f"sum{rank}.npy"), np.array(out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_rank_ordered_scalar_sum(tmp_path):
    """Scalars are summed in rank order on every rank: identical bits everywhere."""
    import torch.multiprocessing as mp

    world = 3
    mp.spawn(_sum_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    s = [np.load(tmp_path / f"sum{r}.npy") for r in range(world)]
    assert np.array_equal(s[0], s[1]) and np.array_equal(s[1], s[2])
    assert s[0][0] == (0.1 + 0.2) + 0.30000000000000004
    assert s[0][1] == (1e16 + 1.0) + 1.0


def _slab_worker(rank, world, port, outdir):
    """z-slab sharding: rank r owns slices ctk_shard_slabs(nz, G, r); A x partial projections
    are sum-reduced (A x = sum_r A x_r), domain reductions summed in rank order."""
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle.oracle import Restated, bench_geometry
    from paper_2211_14212_b200.comm import TorchComm, shard_slabs

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    orc = Restated()
    g = bench_geometry(12, 10)
    gt = orc.shepp_logan_3d(12, np.float64)
    b = orc.forward(g, gt)
    z0, cnt = shard_slabs(g.nz, world, rank)
    n = g.nx * g.ny
    comm = TorchComm(rank, world, device="cpu")

    def ax(xs):  # this rank's slab operator: the full one on x zero outside the slab
        full = np.zeros(g.domain_size)
        full[z0 * n:(z0 + cnt) * n] = xs
        y = orc.forward(g, full)
        comm.allreduce_buffer(y.ctypes.data, y.size, 1)
        return y

    def atb(y):  # local: the full backprojection restricted to the slab
        return orc.back(g, y)[z0 * n:(z0 + cnt) * n].copy()

    def dnorm(v):
        return np.sqrt(comm.sum_scalar(float(v @ v)))

    k_max = 6
    beta1 = float(np.linalg.norm(b))  # range vectors are replicated
    u = b / beta1
    v = atb(u)
    alpha = dnorm(v)
    v = v / alpha
    w = v.copy()
    x = np.zeros_like(v)
    phibar, rhobar = beta1, alpha
    hist = []
    for _ in range(k_max):
        un = ax(v) - alpha * u
        beta = float(np.linalg.norm(un))
        u = un / beta
        vn = atb(u) - beta * v
        alpha = dnorm(vn)
        v = vn / alpha
        rho = np.hypot(rhobar, beta)
        c, s = rhobar / rho, beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        x = x + (phi / rho) * w
        w = v - (theta / rho) * w
        hist.append((phibar / beta1, float(np.linalg.norm(ax(x) - b)) / beta1))
    np.savez(os.path.join(outdir, f"slab{rank}.npz"), x=x, hist=np.array(hist), z0=z0, cnt=cnt)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_slab_sharded_lsqr_gloo(tmp_path):
    import torch.multiprocessing as mp

    from oracle.oracle import Restated, bench_geometry, lsqr

    world = 3
    mp.spawn(_slab_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"slab{r}.npz") for r in range(world)]
    assert [int(p["z0"]) for p in parts] == [0, 4, 8] and [int(p["cnt"]) for p in parts] == [4, 4, 4]
    # the replicated scalars (residual histories) are bitwise identical on every rank
    assert all(np.array_equal(parts[0]["hist"], p["hist"]) for p in parts)
    orc = Restated()
    g = bench_geometry(12, 10)
    gt = orc.shepp_logan_3d(12, np.float64)
    b = orc.forward(g, gt)
    want = lsqr(lambda v: orc.forward(g, v), lambda v: orc.back(g, v), b, 6, tol=0.0, stop_inc=False)
    x = np.concatenate([p["x"] for p in parts])
    assert np.linalg.norm(x - want["x"]) <= 1e-10 * np.linalg.norm(want["x"])
    assert np.allclose(parts[0]["hist"][:, 1], want["explicit"], rtol=1e-10)
    assert np.allclose(parts[0]["hist"][:, 0], want["implicit"], rtol=1e-10)
