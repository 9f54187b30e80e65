import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2211_14212_b200 as ctk
from oracle.oracle import Reference
from geoms import cone_wide, cone_multitile, to_ctk
R = Reference()
def rel(a, b): return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))
for name, g in (("wide", cone_wide()), ("multitile", cone_multitile())):
    p = ctk.projector_pair(to_ctk(g))
    rng = np.random.default_rng(7)
    for kind in ("absrand_vol_proj", "const_vol_proj", "absrand_proj"):
        if kind == "absrand_proj":
            y = np.abs(rng.standard_normal(g.range_size))
        else:
            x = np.abs(rng.standard_normal(g.domain_size)) if kind.startswith("absrand") else np.ones(g.domain_size)
            y = R.forward(g, x.astype(np.float32).astype(np.float64))
        y = y.astype(np.float32).astype(np.float64)
        print(name, kind, "atb %.3g" % rel(p.apply_back(y.astype(np.float32)), R.back(g, y, 0)), "voxel %.3g" % rel(ctk.projector_pair(to_ctk(g), ctk.BackprojectVariant.voxel_driven).apply_back(y.astype(np.float32)), R.back(g, y, 1)))
