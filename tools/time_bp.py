"""Median device time (ms) of f32 Ax and matched A^T b at the bench geometry (A/B timing of
kernel variants: load one with CTK_B200_LIB=build_variants/NAME/libctk_b200.so)."""
import argparse, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512); ap.add_argument("--angles", type=int, default=360)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--projector", default="joseph", choices=["joseph", "siddon"])
a = ap.parse_args()
g = ctk.bench_geometry(a.n, a.angles)
p = ctk.projector_pair(g, projector=getattr(ctk.ProjectorKind, a.projector))
x = ctk.shepp_logan_3d(a.n)
y = torch.empty(p.range_size, device="cuda")
xb = torch.empty_like(x)
out = {}
for name, fn in (("ax", lambda: p.forward(x, y)), ("atb", lambda: p.back(y, xb))):
    ts = []
    for _ in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name] = round(statistics.median(ts[1:]), 3)
print(os.environ.get("CTK_B200_LIB", "default"), a.projector, out, "checksum", float(xb.double().sum()))
