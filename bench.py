#!/usr/bin/env python
"""Benchmark of the B200 Ax / A^T b hot path (BASELINE.json metric).

Workload (config 3 of BASELINE.json, the shape the metric is quoted on): LSMR with
Tikhonov damping lambda = 30, 50 iterations, 512^3 Shepp-Logan volume (device-rasterised,
h = 1), 512^2 detector, 360 equidistant angles, cone beam DSO = 2n, DOD = n, pixel 1.5,
matched backprojector, fp32 data.  One STEP = one full solve (50 Krylov iterations, each
= 2 Ax + 1 A^T b + fused BLAS-1, explicit residual included, as the reference does).
`value` = Krylov iterations/s of the whole job; Ax / A^T b Gray-voxel/s are reported too.

Multi-GPU (torchrun): angles are sharded contiguously across ranks, the volume replicated;
A^T b partial volumes are sum-reduced with NCCL and range dots summed in rank order.

--impl reference: times the reference CPU implementation (oracle/_ref, the unmodified
reference headers compiled here) on the host cores, on a bounded sample of the same
workload (Ax + matched A^T b over a subset of angles, extrapolated to iterations/s).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Krylov iters/s + Ax/Atb Gray-voxel/s, 512^3 vol, 512^2 det, 360 angles"
GATHER_BYTES_PER_SAMPLE = 16  # 4 fp32 taps per bilinear sample


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--config", default=None, choices=["C1", "C2", "C3", "C4", "C5"],
                   help="BASELINE.json config preset (default: C3, the headline metric's config)")
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=512)
    p.add_argument("--angles", type=int, default=360)
    p.add_argument("--iters", type=int, default=50)
    p.add_argument("--lam", type=float, default=30.0)
    p.add_argument("--solver", default="lsmr", choices=["lsmr", "lsqr", "cgls", "hybrid_lsqr", "cgls_tv"],
                   help="lsmr (C3, the headline), lsqr (C2), cgls (C1), hybrid_lsqr GCV (C4), cgls_tv (C5)")
    p.add_argument("--outer", type=int, default=4, help="cgls_tv outer (reweighting) cycles")
    p.add_argument("--projector", default="joseph", choices=["joseph", "siddon"],
                   help="joseph (C1, C3) or siddon (C2: exact-length projector and its transpose)")
    p.add_argument("--shard", default="angle", choices=["angle", "slab"],
                   help="multi-GPU partition (SURVEY.md 8(e)): angle blocks (C3/C4) or z-slabs (C5)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=20.0, help="unused (kept for old command lines)")
    a = p.parse_args()
    if a.config:
        a.__dict__.update(CONFIGS[a.config])
    return a


# BASELINE.json configs; every preset is the named acquisition at its full size
CONFIGS = {
    "C1": dict(solver="cgls", n=64, angles=100, iters=20, projector="joseph", shard="angle"),
    "C2": dict(solver="lsqr", n=256, angles=180, iters=50, projector="siddon", shard="angle"),
    "C3": dict(solver="lsmr", n=512, angles=360, iters=50, lam=30.0, projector="joseph", shard="angle"),
    "C4": dict(solver="hybrid_lsqr", n=512, angles=720, iters=50, projector="joseph", shard="angle"),
    # C5: 4 outer x 15 inner; lambda from the coarse 128^3 proxy sweep (tools/tv_lambda_sweep.py)
    "C5": dict(solver="cgls_tv", n=1024, angles=1600, iters=60, outer=4, lam=0.1, projector="joseph", shard="slab"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def traffic_bytes(kernel, n, na):
    """DRAM bytes per operation of the dominant kernel from the committed ncu capture (same
    workload only), else None."""
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02")
    for name in ("traffic_ax_512_360.json", "traffic_atb_512_360.json", "traffic_ax2_512_360.json"):
        try:
            with open(os.path.join(here, name)) as f:
                t = json.load(f)
        except (OSError, ValueError):
            continue
        if t.get("kernel") == kernel and t.get("n") == n and t.get("angles") == na:
            return t["dram_bytes_per_op"]  # bytes per operation (compare "algorithmic_bytes")
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def window(self, t0, t1):
        """Keep only the samples taken inside the timed region [t0, t1]."""
        self.lines = [(t, ln) for t, ln in self.lines if t0 <= t <= t1]

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample_angles(n, na, cores):
    """The CPU sample: 64 evenly spaced angles up to 512^3 (16 at 1024^3, one
    per host thread, where one angle is 8x the work), never fewer than the thread count."""
    return min(na, max(cores, 64 if n <= 512 else 16))


def cpu_reference_rate(n, na, reps=3, dtype_f32=True):
    """Reference CPU path (oracle/_ref) on the host cores: Ax + matched A^T b over an evenly
    spaced subset of S angles, best of `reps` runs after one warm-up, extrapolated linearly in
    angles (projector.hpp:150,187 are independent per angle) to one Krylov iteration = 2 Ax +
    1 A^T b (BLAS-1, CGS2 and the TV stencils excluded, which favours the CPU)."""
    import numpy as np

    from oracle.oracle import Reference, Restated, bench_geometry

    kind = "reference" if Reference.available() else "port"
    cores = os.cpu_count() or 1
    # the reference's matched A^T b keeps one partial volume per thread (projector.hpp:172-201):
    # cap the threads so those stay within ~40 % of the free host memory
    try:
        import psutil

        free = psutil.virtual_memory().available
        per = (4 if dtype_f32 else 8) * float(n) ** 3
        cores = max(1, min(cores, int(0.4 * free / per) - 1))
    except Exception:
        pass
    orc = Reference() if kind == "reference" else None
    if orc is not None:
        orc.set_threads(cores)
    rest = Restated()
    g = bench_geometry(n, na)
    dt = np.float32 if dtype_f32 else np.float64
    x = rest.shepp_logan_3d(n, dt)
    S = cpu_sample_angles(n, na, cores)
    gs = g.subset(np.linspace(0, na, S, endpoint=False).astype(int))

    def run():
        t0 = time.perf_counter()
        y = orc.forward(gs, x) if orc else rest.forward(gs, x)
        t1 = time.perf_counter()
        _ = orc.back(gs, y, 0) if orc else rest.back(gs, y)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    run()  # warm-up (threads, page faults)
    best = min((run() for _ in range(max(1, reps))), key=lambda t: t[0] + t[1])
    tax, tbt = best
    t_iter = (na / S) * (2.0 * tax + tbt)
    samples_ax = S * n * n * n  # rays*slices for S angles (Gray-voxel normaliser)
    return {
        "iters_per_s": 1.0 / t_iter,
        "ax_gvox_s": 1e-9 * samples_ax / tax,
        "atb_gvox_s": 1e-9 * samples_ax / tbt,
        "kind": kind,
        "cores": cores,
        "sample": f"Ax + matched A^T b on {S} of {na} evenly spaced angles, best of {max(1, reps)} after a warm-up "
                  f"({'f32' if dtype_f32 else 'f64'}, reference headers -O3 -fopenmp, {cores} threads), "
                  f"extrapolated x{na / S:.1f} to 2 Ax + 1 A^T b per iteration",
        "seconds": tax + tbt,
    }


def reference_arm(args, rank, world):
    """The reference's own CPU implementation on this box's host cores, timed on the same
    sample as bench's cpu_baseline: each timed step is one best-of-1 run of the Ax + A^T b
    sample (one warm-up first); at most 3 timed steps so the run stays within minutes."""
    if rank != 0:
        return
    steps = max(1, min(args.steps, 3))
    vals, last = [], None
    for i in range(steps):
        r = cpu_reference_rate(args.n, args.angles, reps=1)
        vals.append(r["iters_per_s"])
        last = r
    v = max(vals)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": "iters/s",
        "n_gpus": args.gpus,
        "steps": steps,
        "warmup": 1,
        "ms_per_step": 1000.0 / v,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic Shepp-Logan 3D (phantom.hpp), b = A x",
        "config": {"workload": workload_desc(args) + "; CPU sample extrapolated"},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"] + f"; best of {steps} steps"},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "ax_gvox_s": last["ax_gvox_s"],
        "atb_gvox_s": last["atb_gvox_s"],
    }
    print(json.dumps(line), flush=True)


def config_name(args):
    for k, c in CONFIGS.items():
        if all(getattr(args, f) == v for f, v in c.items() if f != "shard"):
            return f"BASELINE config {k[1]}"
    return "custom"


def workload_desc(args):
    n, na = args.n, args.angles
    sd = {"lsmr": f"LSMR lambda={args.lam}", "hybrid_lsqr": "hybrid LSQR (GCV, CGS2 reorthogonalisation)",
          "cgls_tv": f"IRN-TV-CGLS {args.outer} outer x {args.iters // max(1, args.outer)} inner, lambda={args.lam}"
          }.get(args.solver, args.solver.upper())
    return (f"{sd}, {args.iters} iters/step, {n}^3 volume, {n}^2 detector, {na} angles, cone DSO=2n DOD=n pixel 1.5, "
            f"matched {args.projector.capitalize()} ({config_name(args)})")


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import numpy as np
    import torch

    import paper_2211_14212_b200 as ctk
    from paper_2211_14212_b200.comm import NcclComm, shard_angles, shard_slabs

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    n, na = args.n, args.angles
    full = ctk.bench_geometry(n, na)
    proj_kind = ctk.ProjectorKind.siddon if args.projector == "siddon" else ctk.ProjectorKind.joseph

    def solve(bb):
        if args.solver == "lsmr":
            return ctk.lsmr(pair, bb, args.lam, opts)
        if args.solver == "hybrid_lsqr":
            return ctk.hybrid_lsqr(pair, bb, ctk.HybridStrategy.gcv(), opts)
        if args.solver == "cgls_tv":
            return ctk.cgls_tv(pair, bb, args.lam, args.outer, args.iters // args.outer, opts)
        return getattr(ctk, args.solver)(pair, bb, opts)
    # synthetic inputs, resident in HBM: phantom rasterised on the device, b = A x
    x_true = ctk.shepp_logan_3d(n)
    comm = NcclComm(rank, world) if world > 1 else None
    if args.shard == "slab":
        # z-slab with the band-sharded range: this rank's slices of x and its
        # detector-row window of b; b from the whole-volume operator (setup, not timed)
        z0, nzl = shard_slabs(n, world, rank)
        b = torch.empty(ctk.projector_pair(full).range_size, dtype=torch.float32, device="cuda")
        ctk.projector_pair(full).forward(x_true, b)
        x_true = x_true[z0 * n * n:(z0 + nzl) * n * n].contiguous()
        pair = ctk.projector_pair(full, slab=(z0, nzl), projector=proj_kind, comm=comm, shard_range=comm is not None)
        if comm is not None:
            b = pair.projector.local_range(b).contiguous()
    else:
        first, count = shard_angles(na, world, rank)
        pair = ctk.projector_pair(full.subset(first, count), projector=proj_kind, comm=comm)
        b = torch.empty(pair.range_size, dtype=torch.float32, device="cuda")
        pair.forward(x_true, b)
    proj = pair.projector
    torch.cuda.synchronize()
    opts = ctk.SolverOptions(max_iters=args.iters, stop_on_explicit_residual_increase=False, residual_tolerance=0.0)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def maxed(t):
        if dist is None:
            return t
        v = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    # ---- per-kernel timing (CUDA events recorded by the library around its main kernel, on
    # the stream that kernel runs on), 3 repeats each, inputs > L2 (512 MiB volume)
    y = torch.empty_like(b)
    xb = torch.empty_like(x_true)
    ax_ms, bt_ms, ax_call_ms = [], [], []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pair.forward(x_true, y)
        e1.record()
        torch.cuda.synchronize()
        ax_ms.append(proj.last_kernel_ms())
        ax_call_ms.append(e0.elapsed_time(e1))
        pair.back(y, xb)
        torch.cuda.synchronize()
        bt_ms.append(proj.last_kernel_ms())
    t_ax = statistics.median(ax_ms[1:])
    t_bt = statistics.median(bt_ms[1:])
    # the two-volume march the solvers run once per iteration (the explicit residual's A x
    # with the next A v or A p; every bench solver on a whole-volume handle)
    t_pair = None
    if args.solver in ("lsqr", "lsmr", "hybrid_lsqr", "cgls", "cgls_tv") and not (args.shard == "slab" and world > 1) \
            and os.environ.get("CTK_FWD_NO_PAIR") != "1":
        y2 = torch.empty_like(b)
        pair_ms = []
        for _ in range(4):
            proj.forward_pair(x_true, y, xb, y2)
            torch.cuda.synchronize()
            pair_ms.append(proj.last_kernel_ms())
        t_pair = statistics.median(pair_ms[1:])
        del y2

    # ---- the solve: W warmup steps, K timed steps (device-resident b and x).  The clock
    # sampler starts before the warmup so its start-up never overlaps the timed region.
    # A window that saw a hardware or thermal slowdown is re-measured once (timing rules).
    remeasured = False
    for attempt in range(2):
        with Clocks(local) as clk:
            for _ in range(args.warmup if attempt == 0 else 1):
                solve(b)
            barrier()
            launches0 = ctk.launch_count()
            t0 = time.perf_counter()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            runs = []
            for _ in range(args.steps):
                res = solve(b)
                runs.append(res.iterations_run)
            s1.record()
            barrier()
            t1 = time.perf_counter()
            wall = t1 - t0
            launches = ctk.launch_count() - launches0
        clk.window(t0, t1)
        throttled = bool(set(clk.summary().get("reasons", [])) &
                         {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"})
        if dist is not None:  # every rank takes the same decision
            flag = torch.tensor([1.0 if throttled else 0.0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            throttled = bool(flag.item())
        if not throttled or attempt == 1:
            break
        remeasured = True
    dev_ms = maxed(s0.elapsed_time(s1))
    # every timed solve must have run all its iterations (no early stop inflating the rate)
    assert all(r == args.iters for r in runs), f"iterations_run {runs} != {args.iters}"
    iters_total = sum(runs)
    free_b, total_b = torch.cuda.mem_get_info()  # device-wide: sees the library's own cudaMalloc
    ms_per_step = dev_ms / args.steps
    value = iters_total / (dev_ms / 1000.0)

    # ---- end-to-end through the public API with HOST (pinned) buffers
    b_host = torch.empty(pair.range_size, dtype=torch.float32, pin_memory=True)
    b_host.copy_(b.cpu())
    b_np = b_host.numpy()
    e2e_steps = max(1, min(args.steps, 2))
    with Clocks(local) as clk_e2e:
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r = solve(b_np)  # H2D b, solve, D2H x inside the call
        barrier()
        t1 = time.perf_counter()
    clk_e2e.window(t0, t1)
    e2e_s = maxed(t1 - t0)
    e2e_value = args.iters * e2e_steps / e2e_s
    assert r.iterations_run == args.iters

    hbm_peak, sm_mhz, peak_src = peaks()
    # this rank's share of the work: its angle block (angle) or its slab of slices (slab)
    my_angles = count if args.shard == "angle" else na
    my_slices = n if args.shard == "angle" else nzl
    nvox, nproj = n * n * my_slices, my_angles * n * n
    samples = my_angles * n * n * my_slices  # Gray-voxel normaliser (rays x slices)
    ax_gvox = 1e-9 * samples / (t_ax / 1e3)
    bt_gvox = 1e-9 * samples / (t_bt / 1e3)
    # per iteration: A^T b once, and either two forward marches or one two-volume march
    if t_pair is None:
        share_ax, share_bt = 2 * t_ax, t_bt
        dom = "k_ax_f32" if share_ax >= share_bt else "k_atb_matched_f32"
        t_dom = t_ax if dom == "k_ax_f32" else t_bt
        vols = 1
    else:
        dom = "k_ax2_f32" if t_pair >= t_bt else "k_atb_matched_f32"
        t_dom = t_pair if dom == "k_ax2_f32" else t_bt
        vols = 2 if dom == "k_ax2_f32" else 1
    alg_bytes = 4.0 * (nvox + nproj) * vols
    achieved = alg_bytes / (t_dom / 1e3) / 1e9
    gather_peak_arith = 148 * 128 * sm_mhz * 1e6 / GATHER_BYTES_PER_SAMPLE / 1e9  # G samples/s at 128 B/clk/SM
    gather_peak, gather_src = gather_peak_arith, "arithmetic: 16 B/sample at 128 B/clk/SM x 148 SMs"
    try:  # the measured ceiling: tools/gather_peak.cu, the Ax sample's four tap loads on L1-resident data
        for ln in open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02", "gather_peak.json")):
            d = json.loads(ln)
            if d.get("pattern") == "ax4":
                gather_peak = d["samples_per_s"] / 1e9
                gather_src = ("measured: tools/gather_peak.cu ax4 (the Ax sample's 4 tap loads, L1-resident, "
                              "profiles/r02/gather_peak.json); arithmetic 128 B/clk/SM ceiling "
                              f"{gather_peak_arith:.0f} G samples/s")
    except (OSError, ValueError, KeyError):
        pass
    vol_mib, proj_mib = 4 * nvox / 2**20, 4 * nproj / 2**20
    l2_note = (f"inputs larger than L2 (volume {vol_mib:.0f} MiB, projections {proj_mib:.0f} MiB)"
               if min(vol_mib, proj_mib) > 126 else
               f"inputs fit in L2 (volume {vol_mib:.0f} MiB, projections {proj_mib:.0f} MiB); no flush between "
               f"iterations -- not a headline size")
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "iters/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic: Shepp-Logan 3D rasterised on device (phantom.hpp), b = A x (GPU Ax)",
        "config": {"workload": workload_desc(args),
                   "parallelism": f"{args.shard}-sharded x{world}" if world > 1 else "single GPU",
                   "l2": l2_note},
        "ax_gvox_s": ax_gvox,
        "atb_gvox_s": bt_gvox,
        "kernels_ms": {"k_ax_f32": t_ax, "k_atb_matched_f32": t_bt, "k_ax2_f32": t_pair,
                       "ax_call": statistics.median(ax_call_ms[1:])},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic_bytes(dom, n, my_angles) if my_slices == n else None, "algorithmic_bytes": alg_bytes,
                     "note": f"algorithmic bytes 4*(N_vox+N_proj) per launch; peak {peak_src}; traffic = measured "
                             "DRAM bytes of the same operation (both slice-chunk launches) from the committed ncu "
                             "capture, profiles/r02/traffic_{ax,atb}_512_360.json, when the workload matches; the volume "
                             "slab of each detector-row band is re-read from DRAM by design (L2 residency per band; "
                             "8.4 GB per Ax at C3 = 176 GB/s, 2.7 % of HBM: the kernel is bound on chip)"},
        "roofline_gather": {"kernel": dom, "achieved": vols * samples / (t_dom / 1e3) / 1e9, "peak": gather_peak,
                            "unit": "G samples/s", "frac": vols * samples / (t_dom / 1e3) / 1e9 / gather_peak,
                            "note": "binding on-chip ceiling (SURVEY.md 8(d)), " + gather_src +
                                    ("; k_ax2_f32 = the two-volume march (two samples per ray-slice, one per volume)"
                                     if vols == 2 else "")},
        "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": 4 * nproj, "d2h_bytes_per_step": 4 * nvox,
                "clocks": clk_e2e.summary()},
        "gpu_launches": launches,
        "clocks": dict(clk.summary(), remeasured=remeasured),
        "wall_s_timed": wall,
        "final_explicit_residual": res.log.explicit_residual[-1],
        "device_mem_used_gib": (total_b - free_b) / 2**30,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_reference_rate(n, na, reps=3)
            line["cpu_baseline"] = {"value": cb["iters_per_s"], "unit": "iters/s", "cores": cb["cores"],
                                    "kind": cb["kind"],
                                    "sample": cb["sample"] + ("; the reference has no Siddon projector, so its Joseph "
                                                              "path (same rays and sizes) stands in"
                                                              if args.projector == "siddon" else ""),
                                    "ax_gvox_s": cb["ax_gvox_s"],
                                    "atb_gvox_s": cb["atb_gvox_s"]}
        except Exception as e:  # reported, never fatal to the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "iters/s", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
