"""One timed solve of a BASELINE config on one GPU (the configs bench.py does not default to):
  C4: hybrid LSQR, GCV, reorth, 50 iterations, 512^3, 512^2, 720 views
  C5: CGLS-TV (IRN), 4 outer x 15 inner, 1024^3, 1024^2, 1600 views (z-slab sharding at 8
      GPUs; one GPU holds the whole volume here)
A short warm-up solve precedes the timed one; device time with CUDA events."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk

ap = argparse.ArgumentParser()
ap.add_argument("--config", choices=["C4", "C5"], required=True)
ap.add_argument("--n", type=int, default=0); ap.add_argument("--angles", type=int, default=0)
ap.add_argument("--iters", type=int, default=50)
# C5 TV weight from the 128^3 proxy sweep (tools/tv_lambda_sweep.py: 0.1); the cost per
# iteration does not depend on it (the 1024^3 run in DESIGN.md used 0.5)
ap.add_argument("--tv-lam", type=float, default=0.1)
a = ap.parse_args()
n = a.n or (512 if a.config == "C4" else 1024)
na = a.angles or (720 if a.config == "C4" else 1600)
g = ctk.bench_geometry(n, na)
pair = ctk.projector_pair(g)
x = ctk.shepp_logan_3d(n)
b = torch.empty(pair.range_size, device="cuda")
pair.forward(x, b)
del x
torch.cuda.synchronize()

def run(iters, outer=4, inner=15):
    opts = ctk.SolverOptions(max_iters=iters, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)
    if a.config == "C4":
        return ctk.hybrid_lsqr(pair, b, ctk.HybridStrategy.gcv(), opts), iters
    return ctk.cgls_tv(pair, b, a.tv_lam, outer, inner, opts), outer * inner

run(2, 1, 2)  # warm-up: workspaces, tables, clocks
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res, k = run(a.iters)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"config": a.config, "n": n, "angles": na, "iterations": k, "ms": ms, "iters_per_s": k / (ms / 1e3),
                  "final_explicit_residual": res.log.explicit_residual[-1],
                  "stored_bases": [res.stored_domain_basis, res.stored_range_basis],
                  "peak_mem_gib": torch.cuda.max_memory_allocated() / 2**30}))
