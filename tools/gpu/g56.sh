# C3 launch list (5-iteration LSMR) and the C5 bench line
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_pair.csv python tools/solve_once.py --n 512 --angles 360 --iters 5 --reps 1 > gpurun_out/g56_ncu.log 2>&1; tail -1 gpurun_out/g56_ncu.log
python tools/launch_agg.py gpurun_out/launches_c3_pair.csv > gpurun_out/launch_shares_c3_pair.txt; head -12 gpurun_out/launch_shares_c3_pair.txt
timeout 2700 python bench.py --config C5 --steps 1 --warmup 3 > gpurun_out/g56_c5.json 2> gpurun_out/g56_c5.err; tail -c 300 gpurun_out/g56_c5.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/g56_c5.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("kernels_ms"), d["clocks"]["reasons"], d.get("device_mem_used_gib"))
P
