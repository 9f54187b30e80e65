"""The native NCCL communicator (libnccl.so.2 dlopen'd by libctk_b200.so) on the one GPU
this harness has: a world-size-1 NCCL communicator drives every collective call of the
angle-sharded and z-slab solver paths for real (the all-reduce of A^T b, the projection
all-reduce and halo exchange of slab mode, the rank-ordered scalar gathers), and the solves
must reproduce the communicator-free ones.  Multi-rank behaviour is covered on CPU by
tests/test_sharding_gloo.py; ranks that wait on each other are never run on one GPU."""
import os
import socket
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, %r)
    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200.comm import NcclComm

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    comm = NcclComm(0, 1)
    n, na = 32, 24
    g = ctk.bench_geometry(n, na)
    x = ctk.shepp_logan_3d(n)
    ref_pair = ctk.projector_pair(g)
    b = ref_pair.apply_forward(x)
    opts = ctk.SolverOptions(max_iters=5, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)

    def rel(a, c):
        a, c = a.double().cpu(), c.double().cpu()
        return float((a - c).norm() / c.norm())

    for solver in ("lsqr", "cgls"):
        r0 = getattr(ctk, solver)(ref_pair, b, opts)
        for slab in (None, (0, n)):
            p = ctk.projector_pair(g, slab=slab)
            p.projector.attach_comm(comm)
            r1 = getattr(ctk, solver)(p, b, opts)
            e = rel(r1.x, r0.x)
            assert e < 1e-6, (solver, slab, e)
            assert np.allclose(r1.log.explicit_residual, r0.log.explicit_residual, rtol=1e-6, atol=0)
            print(solver, slab, "rel", e)
    t0 = ctk.cgls_tv(ref_pair, b, 0.05, 2, 3, opts)
    p = ctk.projector_pair(g, slab=(0, n))
    p.projector.attach_comm(comm)
    t1 = ctk.cgls_tv(p, b, 0.05, 2, 3, opts)
    e = rel(t1.x, t0.x)
    assert e < 1e-6, ("cgls_tv", e)
    print("cgls_tv slab rel", e)
    # band-sharded range over the NCCL communicator (one rank owns every row)
    p = ctk.projector_pair(g, slab=(0, n), comm=comm, shard_range=True)
    assert p.projector.range_rows() == (0, g.nv, 0, g.nv)
    t2 = ctk.cgls_tv(p, b, 0.05, 2, 3, opts)
    e = rel(t2.x, t0.x)
    assert e < 1e-6, ("cgls_tv band", e)
    print("cgls_tv band rel", e)
    del comm
    dist.destroy_process_group()
    print("NCCL_OK")
""") % ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_nccl_world1_solves_match():
    env = {**os.environ, "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(_free_port())}
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "NCCL_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
