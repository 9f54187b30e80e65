"""Debug helper: f32 Ax / matched A^T b at the bench geometry, one call each, reporting failures.
python tools/dbg_sid.py N ANGLES joseph|siddon ax|atb ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2211_14212_b200 as ctk

n, na, proj = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
g = ctk.bench_geometry(n, na)
p = ctk.projector_pair(g, dtype="float32", projector=getattr(ctk.ProjectorKind, proj))
x = ctk.shepp_logan_3d(n)
for what in sys.argv[4:]:
    try:
        if what == "ax":
            y = p.apply_forward(x)
            torch.cuda.synchronize()
            print(proj, "ax ok", float(y.sum()))
        else:
            y = torch.ones(p.range_size, device="cuda")
            xb = p.apply_back(y)
            torch.cuda.synchronize()
            print(proj, "atb ok", float(xb.sum()))
    except Exception as e:
        print(proj, what, "FAILED", str(e)[:300])
        break
