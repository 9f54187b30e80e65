"""One Siddon Ax + exact transpose at the C2 geometry (256^3, 256^2, 180 views) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_14212_b200 as ctk  # noqa: E402

n, na = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (256, 180)
g = ctk.bench_geometry(n, na)
p = ctk.projector_pair(g, projector=ctk.ProjectorKind.siddon)
x = ctk.shepp_logan_3d(n)
y = torch.empty(p.range_size, device="cuda")
p.forward(x, y)
xb = torch.empty_like(x)
p.back(y, xb)
torch.cuda.synchronize()
print("ok")
