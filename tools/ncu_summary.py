"""One-page summary of a single-kernel ncu --set full report (ncu -i REP --page raw --csv):
the metrics quoted in DESIGN.md plus the pc-sampling stall histogram."""
import csv
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "sm__inst_executed.avg.per_cycle_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
           "launch__block_size", "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]

rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, vals = rows[0], rows[1], rows[2]
col = {n: i for i, n in enumerate(h)}
if title:
    print("# " + title)
print(f"{'Kernel Name':70s} {vals[col['Kernel Name']]}")
for m in METRICS:
    if m in col:
        print(f"{m:70s} {vals[col[m]]} {units[col[m]]}")
print("warp stall samples (pc sampling):")
pre = "smsp__pcsamp_warps_issue_stalled_"
for n in h:
    if n.startswith(pre) and not n.endswith("_not_issued"):
        v = vals[col[n]].replace(",", "")
        if v and float(v) > 0:
            print(f"    {n[len(pre):]} {v}")
