"""GPU timeline of a short solve (torch.profiler / CUPTI sees every kernel in the process):
per-kernel totals and the idle gaps between consecutive kernels."""
import argparse, collections, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_14212_b200 as ctk

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512); ap.add_argument("--angles", type=int, default=360)
ap.add_argument("--iters", type=int, default=5); ap.add_argument("--out", default="gpurun_out/timeline.json")
a = ap.parse_args()
g = ctk.bench_geometry(a.n, a.angles); pair = ctk.projector_pair(g)
x = ctk.shepp_logan_3d(a.n); b = torch.empty(pair.range_size, device="cuda"); pair.forward(x, b)
opts = ctk.SolverOptions(max_iters=a.iters, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)
ctk.lsmr(pair, b, 30.0, opts); torch.cuda.synchronize()  # warm: workspaces allocated
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    ctk.lsmr(pair, b, 30.0, opts); torch.cuda.synchronize()
prof.export_chrome_trace(a.out)
ev = [e for e in json.load(open(a.out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
tot = collections.defaultdict(float); cnt = collections.Counter()
for e in ev:
    tot[e["name"][:60]] += e["dur"]; cnt[e["name"][:60]] += 1
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
busy = sum(e["dur"] for e in ev)
print(f"span {span/1e3:.1f} ms, busy {busy/1e3:.1f} ms, idle {(span-busy)/1e3:.1f} ms over {len(ev)} ops")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {k:60s} {cnt[k]:4d} {v/1e3:9.2f} ms")
gaps = sorted(((ev[i+1]["ts"] - (ev[i]["ts"] + ev[i]["dur"]), ev[i]["name"][:40], ev[i+1]["name"][:40]) for i in range(len(ev)-1)), reverse=True)
print("largest gaps (us):")
for gp in gaps[:12]: print(f"  {gp[0]:10.1f}  after {gp[1]}  before {gp[2]}")
