"""Small operator and solver cases for compute-sanitizer (tests/test_gpu_sanitizer.py):
f32 Joseph Ax (slice-chunked and z-slab), matched A^T b through the plane backprojector (the
128- or 256-row tile, chosen by CTK_BP_TILE), voxel-driven A^T b, the exact f64 kernels, the
Siddon pair, and two LSQR / CGLS-TV iterations (BLAS-1, stencils).  Geometries are tiny so
racecheck finishes in seconds; cone_steep adds z-dominant rays, cone_multitile ragged tiles and
bands."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import paper_2211_14212_b200 as ctk
from geoms import cone_default, cone_multitile, cone_steep, parallel3d, to_ctk

rng = np.random.default_rng(0)
what = sys.argv[1] if len(sys.argv) > 1 else "all"
for name, mk in (("cone_default", lambda: cone_default(16, 6)), ("cone_steep", cone_steep), ("parallel3d", parallel3d),
                 ("cone_multitile", cone_multitile)):
    g = to_ctk(mk())
    if name == "cone_multitile":
        g.angles = g.angles[:3]
    for dt in ("float32", "float64"):
        tdt = getattr(torch, dt)
        for proj in (ctk.ProjectorKind.joseph, ctk.ProjectorKind.siddon):
            if what not in ("all", proj.name):
                continue
            if name == "cone_multitile" and (dt == "float64" or proj != ctk.ProjectorKind.joseph):
                continue
            for v in (ctk.BackprojectVariant.matched, ctk.BackprojectVariant.voxel_driven):
                p = ctk.projector_pair(g, v, dtype=dt, projector=proj)
                x = torch.from_numpy(rng.standard_normal(p.domain_size)).to(tdt).cuda()
                y = torch.from_numpy(rng.standard_normal(p.range_size)).to(tdt).cuda()
                p.apply_forward(x)
                p.apply_back(y)
        torch.cuda.synchronize()
    print("operators ok", name, flush=True)
if what in ("all", "joseph"):
    g = to_ctk(cone_default(16, 6))
    # z-slab pair: slices [5, 12) of 16
    ps = ctk.projector_pair(g, slab=(5, 7))
    ps.apply_forward(torch.ones(ps.domain_size, device="cuda"))
    ps.apply_back(torch.ones(ps.range_size, device="cuda"))
    p = ctk.projector_pair(g)
    b = p.apply_forward(ctk.shepp_logan_3d(16))
    ctk.lsqr(p, b, ctk.SolverOptions(max_iters=2))
    ctk.cgls_tv(p, b, 0.1, 1, 2, ctk.SolverOptions(max_iters=2))
    ctk.hybrid_lsqr(p, b, ctk.HybridStrategy.gcv(), ctk.SolverOptions(max_iters=3))
    torch.cuda.synchronize()
    print("solvers ok", flush=True)
print("launches", ctk.launch_count())
