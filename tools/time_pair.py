"""Time the two-volume forward march (Projector.forward_pair) against two forward() calls,
and check the outputs bit for bit.  Usage: time_pair.py [--n 512] [--angles 360]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512); ap.add_argument("--angles", type=int, default=360)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
g = ctk.bench_geometry(a.n, a.angles)
pair = ctk.projector_pair(g)
P = pair.projector
x1 = ctk.shepp_logan_3d(a.n)
x2 = torch.randn_like(x1)
y1 = torch.empty(pair.range_size, device="cuda"); y2 = torch.empty_like(y1)
z1 = torch.empty_like(y1); z2 = torch.empty_like(y1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def tm(f):
    best = 1e30
    for r in range(a.reps + 1):
        torch.cuda.synchronize(); e0.record(); f(); e1.record(); torch.cuda.synchronize()
        if r: best = min(best, e0.elapsed_time(e1))
    return best
t2 = tm(lambda: (pair.forward(x1, z1), pair.forward(x2, z2)))
tp = tm(lambda: P.forward_pair(x1, y1, x2, y2))
same = bool(torch.equal(y1, z1) and torch.equal(y2, z2))
print(f"n={a.n} views={a.angles}: two forward {t2:.2f} ms, pair {tp:.2f} ms ({tp / t2 * 2:.3f} x one forward), bitwise {same}")
