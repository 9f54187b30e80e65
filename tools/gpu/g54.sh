# pair: tests (Joseph + Siddon), DRAM traffic + full ncu of k_ax2, C3 and C2 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd_pair.py tests/test_gpu_siddon.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/g54_c3.json 2> gpurun_out/g54_c3.err
timeout 600 python bench.py --config C2 --steps 3 --warmup 3 > gpurun_out/g54_c2.json 2> gpurun_out/g54_c2.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_ax2_zfast -c 2 --csv --log-file gpurun_out/ncu_traffic_ax2_512.csv python tools/time_pair.py --n 512 --angles 360 --reps 1 > gpurun_out/g54_tr.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ax2_zfast -c 1 -f -o gpurun_out/ax2_512_m6 python tools/time_pair.py --n 512 --angles 360 --reps 1 > gpurun_out/g54_ncu.log 2>&1
python - <<'P'
import json
for f in ["g54_c3", "g54_c2"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("kernels_ms"), d["clocks"]["reasons"], d["roofline"]["kernel"], d["roofline_gather"]["frac"])
    except Exception as e:
        print(f, "ERR", e)
P
tail -2 gpurun_out/g54_ncu.log
