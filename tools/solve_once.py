"""One short LSMR solve on the bench geometry (for launch lists / tracing)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=int, default=256); ap.add_argument("--angles", type=int, default=180)
ap.add_argument("--iters", type=int, default=3); ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
g = ctk.bench_geometry(a.n, a.angles); pair = ctk.projector_pair(g)
x = ctk.shepp_logan_3d(a.n); b = torch.empty(pair.range_size, device="cuda"); pair.forward(x, b); torch.cuda.synchronize()
opts = ctk.SolverOptions(max_iters=a.iters, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)
for r in range(a.reps):
    t0 = time.perf_counter(); res = ctk.lsmr(pair, b, 30.0, opts); torch.cuda.synchronize()
    print(f"solve {a.iters} iters: {(time.perf_counter()-t0)*1e3:.1f} ms")
