"""f32 Ax / matched A^T b vs the reference T=double (oracle/_ref) on RANDOM-SIGNED data --
the worst case for sample-position rounding -- at the config geometries on view subsets:
C3 (512^3 / 512^2) on 4 and 16 of 360 views, C5 (1024^3 / 1024^2) on 4 of 1600 views.
Usage: python tools/precision_signed.py [c3|c5|all]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2211_14212_b200 as ctk
from oracle.oracle import Reference, Geom, CONE3D, equidistant_angles
from geoms import to_ctk


def rel(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def case(R, n, na_total, views, seed=3):
    ang = np.array(equidistant_angles(na_total))[np.linspace(0, na_total - 1, views).astype(int)]
    g = Geom(CONE3D, 2.0 * n, 1.0 * n, 1.5, n, n, n, n, n, 1.0, ang)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(g.domain_size, dtype=np.float32).astype(np.float64)
    y = rng.standard_normal(g.range_size, dtype=np.float32).astype(np.float64)
    p = ctk.projector_pair(to_ctk(g))
    t = time.time(); yr = R.forward(g, x); ta = time.time() - t
    ea = rel(p.apply_forward(torch.from_numpy(x.astype(np.float32)).cuda()), yr)
    del yr
    t = time.time(); br = R.back(g, y, 0); tb = time.time() - t
    eb = rel(p.apply_back(torch.from_numpy(y.astype(np.float32)).cuda()), br)
    print(f"{n}^3 {views}/{na_total} views signed: ax {ea:.3g} atb {eb:.3g} (ref {ta:.1f} s + {tb:.1f} s)", flush=True)
    return ea, eb


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    R = Reference()
    R.set_threads(min(16, os.cpu_count() or 1))
    if which in ("c3", "all"):
        for v in (4, 16):
            case(R, 512, 360, v)
    if which in ("c5", "all"):
        R.set_threads(4)  # per-thread partial volumes of the matched scatter: 8 GiB each at 1024^3
        case(R, 1024, 1600, 4)
