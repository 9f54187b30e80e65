"""f32 Ax / matched A^T b vs the reference T=double at the C3 geometry on a subset of the
360 views (Shepp-Logan phantom, its projections, and random-signed projections)."""
import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2211_14212_b200 as ctk
from oracle.oracle import Reference, Geom, CONE3D, equidistant_angles
from geoms import to_ctk
R = Reference()
def rel(a, b): return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))
n = 512
x = ctk.make_phantom(ctk.PhantomKind.shepp_logan_3d, n, "float64").cpu().numpy()
for nv in [int(v) for v in sys.argv[1:]] or [4, 16]:
    ang = np.array(equidistant_angles(360))[np.linspace(0, 359, nv).astype(int)]
    g = Geom(CONE3D, 2.0 * n, 1.0 * n, 1.5, n, n, n, n, n, 1.0, ang)
    p = ctk.projector_pair(to_ctk(g))
    t = time.time(); yr = R.forward(g, x); ta = time.time() - t
    t = time.time(); br = R.back(g, yr, 0); tb = time.time() - t
    print(nv, "views: phantom ax %.3g atb %.3g (ref %.1f s + %.1f s)" % (
        rel(p.apply_forward(x.astype(np.float32)), yr), rel(p.apply_back(yr.astype(np.float32)), br), ta, tb), flush=True)
