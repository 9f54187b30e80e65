"""Median device time (ms) of the Siddon Ax and exact transpose (f32) at a bench geometry."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk
n, na = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (256, 180)
g = ctk.bench_geometry(n, na)
p = ctk.projector_pair(g, projector=ctk.ProjectorKind.siddon)
x = ctk.shepp_logan_3d(n)
y = torch.empty(p.range_size, device="cuda")
xb = torch.empty_like(x)
out = {}
for name, fn in (("ax", lambda: p.forward(x, y)), ("atb", lambda: p.back(y, xb))):
    ts = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name] = round(statistics.median(ts[1:]), 2)
print(os.environ.get("CTK_B200_LIB", "default"), out, "checksum", float(xb.double().sum()))
