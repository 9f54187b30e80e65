import os, statistics, sys
sys.path.insert(0, '/root/repo')
import torch, paper_2211_14212_b200 as ctk
g = ctk.bench_geometry(256, 180)
p = ctk.projector_pair(g, dtype="float64")
x = ctk.shepp_logan_3d(256, "float64"); y = torch.empty(p.range_size, dtype=torch.float64, device="cuda"); xb = torch.empty_like(x)
p.forward(x, y)
ts = []
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p.back(y, xb); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(os.environ.get("CTK_B200_LIB", "default"), "f64 matched atb", round(statistics.median(ts[1:]), 2), float(xb.sum()))
