"""Device time of Ax / matched A^T b / voxel-driven A^T b for f32 and f64 (and Siddon)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_14212_b200 as ctk

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256); ap.add_argument("--angles", type=int, default=180)
a = ap.parse_args()
g = ctk.bench_geometry(a.n, a.angles)
for dt, tdt in (("float32", torch.float32), ("float64", torch.float64)):
    for proj in (ctk.ProjectorKind.joseph, ctk.ProjectorKind.siddon):
        pm = ctk.projector_pair(g, dtype=dt, projector=proj)
        pv = ctk.projector_pair(g, ctk.BackprojectVariant.voxel_driven, dtype=dt, projector=proj)
        x = ctk.shepp_logan_3d(a.n, dt)
        y = torch.empty(pm.range_size, dtype=tdt, device="cuda")
        xb = torch.empty_like(x)
        res = {}
        for rep in range(2):
            for name, fn in (("ax", lambda: pm.forward(x, y)), ("atb_matched", lambda: pm.back(y, xb)),
                             ("atb_voxel", lambda: pv.back(y, xb))):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record(); torch.cuda.synchronize()
                res[name] = e0.elapsed_time(e1)
        print(dt, proj.name, {k: round(v, 2) for k, v in res.items()})
