"""Device time of f32 Ax / matched A^T b for one z-slab rank's share (default: the C5
acquisition, 1024^3 / 1024^2 / 1600 views, slab 3 of 8) against the whole volume."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk
from paper_2211_14212_b200.comm import shard_slabs

n, na, G, r = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (1024, 1600, 8, 3)))
g = ctk.bench_geometry(n, na)
z0, cnt = shard_slabs(n, G, r)
p = ctk.projector_pair(g, slab=(z0, cnt))
x = ctk.shepp_logan_3d(n)[z0 * n * n:(z0 + cnt) * n * n].contiguous()
y = torch.empty(p.range_size, device="cuda")
xb = torch.empty_like(x)
out = {}
for name, fn in (("ax", lambda: p.forward(x, y)), ("atb", lambda: p.back(y, xb))):
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name] = round(statistics.median(ts[1:]), 1)
print(f"n={n} na={na} slab {r}/{G} = [{z0}, {z0 + cnt})", out)
