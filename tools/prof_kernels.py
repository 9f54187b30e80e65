"""Small driver for ncu: a few Ax / matched A^T b / voxel A^T b launches on the bench
geometry scaled down (default 256^3 volume, 256^2 detector, 180 angles)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--angles", type=int, default=180)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--what", default="ax,atb,vox")
    a = ap.parse_args()
    import torch

    import paper_2211_14212_b200 as ctk

    g = ctk.bench_geometry(a.n, a.angles)
    pair = ctk.projector_pair(g)
    vpair = ctk.projector_pair(g, ctk.BackprojectVariant.voxel_driven)
    x = ctk.shepp_logan_3d(a.n)
    y = torch.empty(pair.range_size, device="cuda")
    xb = torch.empty_like(x)
    pair.forward(x, y)
    for _ in range(a.reps):
        if "ax" in a.what:
            pair.forward(x, y)
            torch.cuda.synchronize()
            print("ax ms", pair.projector.last_kernel_ms())
        if "atb" in a.what:
            pair.back(y, xb)
            torch.cuda.synchronize()
            print("atb ms", pair.projector.last_kernel_ms())
        if "vox" in a.what:
            vpair.back(y, xb)
            torch.cuda.synchronize()
            print("vox ms", vpair.projector.last_kernel_ms())


if __name__ == "__main__":
    main()
