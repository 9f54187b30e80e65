import sys, os
sys.path.insert(0, '/root/repo')
import torch, paper_2211_14212_b200 as ctk
g = ctk.bench_geometry(128, 90)
p = ctk.projector_pair(g, projector=ctk.ProjectorKind.siddon)
x = ctk.shepp_logan_3d(128); y = torch.empty(p.range_size, device="cuda"); p.forward(x, y)
xb = torch.empty_like(x); p.back(y, xb); torch.cuda.synchronize(); print("ok")
