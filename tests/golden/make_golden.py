"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libctkref.so,
built by oracle/Makefile from /root/reference/proj/include).  Run in the container that
has /root/reference:   python tests/golden/make_golden.py
The fixtures are small (< 200 KB) and travel with the repo; nothing reads /root/reference
at test time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Reference  # noqa: E402
from geoms import cone_default, cone_ragged, parallel2d, parallel3d  # noqa: E402

CASES = {
    "parallel2d": lambda: parallel2d(12, 6),
    "parallel3d": lambda: parallel3d(8, 7, 4, 5),
    "cone_default": lambda: cone_default(8, 6),
    "cone_ragged": cone_ragged,
}


def geom_arrays(g):
    return dict(mode=g.mode, dso=g.dso, dod=g.dod, du=g.du, nu=g.nu, nv=g.nv, nx=g.nx, ny=g.ny, nz=g.nz, h=g.h,
                angles=np.asarray(g.angles, dtype=np.float64))


def main():
    ref = Reference()
    ref.set_threads(1)
    for name, mk in CASES.items():
        g = mk()
        rng = np.random.default_rng(20221114)
        x = rng.standard_normal(g.domain_size)
        y = rng.standard_normal(g.range_size)
        y[::5] = 0.0
        out = geom_arrays(g)
        out.update(x=x, y=y, ax=ref.forward(g, x), atb_matched=ref.back(g, y, 0), atb_voxel=ref.back(g, y, 1),
                   ax_f32=ref.forward(g, x.astype(np.float32)))
        b = ref.forward(g, np.abs(x))
        for solver, lam in (("cgls", 0.0), ("lsqr", 0.0), ("lsmr", 3.0)):
            r = ref.solve(g, b, solver, 5, lam=lam, tol=0.0, stop_inc=False)
            out[f"{solver}_x"] = r["x"]
            out[f"{solver}_implicit"] = r["implicit"]
            out[f"{solver}_explicit"] = r["explicit"]
        out["b"] = b
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print("wrote", name)


if __name__ == "__main__":
    main()
