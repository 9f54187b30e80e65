"""C5's TV weight by a coarse sweep on a 128^3 proxy (the reference gives no
value): the C5 acquisition scaled down (DSO = 2n, DOD = n, pixel 1.5, nu = nv = n, views
1600 * 128/1024 = 200), Shepp-Logan phantom scaled to attenuation 0.02/voxel at intensity 2
(line integrals up to ~2, so the count-domain noise NoiseModel{1e5, 0.5, seed 0} is neither
saturated nor negligible), IRN-TV-CGLS 4 x 15; prints the relative error for each lambda and
the best one."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2211_14212_b200 as ctk

n, na = 128, 200
g = ctk.bench_geometry(n, na)
pair = ctk.projector_pair(g)
x = 0.01 * ctk.shepp_logan_3d(n).cpu().numpy()
b = ctk.add_noise(np.maximum(pair.apply_forward(x), 0.0), ctk.NoiseModel(1e5, 0.5, 0))
res = {}
for lam in (0.001, 0.003, 0.01, 0.03, 0.1, 0.3, 1.0):
    opts = ctk.SolverOptions(max_iters=60, stop_on_explicit_residual_increase=False, residual_tolerance=0.0,
                             ground_truth=x)
    r = ctk.cgls_tv(pair, b, lam, 4, 15, opts)
    res[lam] = (r.log.relative_error[-1], min(r.log.relative_error))
    print(f"lambda {lam:g}: final rel. error {res[lam][0]:.4f}, min {res[lam][1]:.4f}", flush=True)
best = min(res, key=lambda k: res[k][0])
print(json.dumps({"proxy": f"{n}^3, {na} views, noisy", "best_lambda": best, "final_rel_error": res[best][0]}))
