"""Wall time of consecutive solves through the device-pointer and the host-pointer entry
points (diagnostic for bench.py's e2e number)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256); ap.add_argument("--angles", type=int, default=180)
ap.add_argument("--projector", default="siddon"); ap.add_argument("--solver", default="lsqr")
a = ap.parse_args()
g = ctk.bench_geometry(a.n, a.angles)
pair = ctk.projector_pair(g, projector=getattr(ctk.ProjectorKind, a.projector))
x = ctk.shepp_logan_3d(a.n); b = torch.empty(pair.range_size, device="cuda"); pair.forward(x, b)
bh = torch.empty(pair.range_size, pin_memory=True); bh.copy_(b.cpu()); bn = bh.numpy()
opts = ctk.SolverOptions(max_iters=50, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)
for kind in ["dev"] * 3 + ["host"] * 3 + ["dev"] * 2:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    bb = b if kind == "dev" else bn
    ctk.lsmr(pair, bb, 30.0, opts) if a.solver == "lsmr" else getattr(ctk, a.solver)(pair, bb, opts)
    torch.cuda.synchronize()
    print(f"{kind} {time.perf_counter() - t0:.3f} s")
