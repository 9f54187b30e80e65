"""Angle sharding through the product's C++ solvers: two
processes on the one GPU, each owning a contiguous angle block (ctk_shard_angles) with the
product's collectives over gloo (host-staged, so no kernel waits on another rank), must
reproduce the unsharded solve for every solver -- the A^T b partial volumes sum-reduced, the
range-space scalars (||u||, CGS2 / Arnoldi coefficients of the range basis, residual norms)
gathered and summed in rank order, so both ranks also hold identical logs and iterates."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SOLVERS = ["cgls", "lsqr", "lsmr", "sirt", "hybrid_lsqr", "ab_gmres", "ba_gmres", "cgls_tv", "flsqr_tv"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from geoms import to_ctk
    from oracle.oracle import Restated, bench_geometry

    orc = Restated()
    g = bench_geometry(24, 16)
    gt = orc.shepp_logan_3d(24, np.float64)
    b = orc.forward(g, gt).astype(np.float32)
    return to_ctk(g), b


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
    import torch.distributed as dist

    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200.comm import TorchComm, shard_angles

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, b = _problem()
    first, count = shard_angles(len(g.angles), world, rank)
    frame = g.nu * g.nv
    bl = b[first * frame:(first + count) * frame].copy()
    comm = TorchComm(rank, world, device="cuda")
    out = {}
    for which in SOLVERS:
        pair = ctk.projector_pair(g.subset(first, count))
        pair.projector.attach_comm(comm)
        r = _solve(ctk, pair, bl, which)
        out[which + "_x"] = r.x
        out[which + "_expl"] = np.array(r.log.explicit_residual)
        out[which + "_impl"] = np.array(r.log.implicit_residual)
        out[which + "_lam"] = np.array(r.log.lambda_)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_angle_sharded_solvers_two_ranks(tmp_path):
    import torch.multiprocessing as mp

    import paper_2211_14212_b200 as ctk

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g, b = _problem()
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for which in SOLVERS:
        ref = _solve(ctk, ctk.projector_pair(g), b, which)
        for key in ("_x", "_expl", "_impl", "_lam"):  # replicated state: bitwise equal on every rank
            assert np.array_equal(ranks[0][which + key], ranks[1][which + key]), which + key
        assert rel_l2(ranks[0][which + "_x"], ref.x) < 1e-4, which
        assert np.allclose(ranks[0][which + "_expl"], ref.log.explicit_residual, rtol=1e-4), which
        assert np.allclose(ranks[0][which + "_impl"], ref.log.implicit_residual, rtol=1e-4), which
