# adopted MINB 6 pair: tests + C3, C4, 45-view share
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fwd_pair.py tests/test_gpu_solvers.py -x -q 2>&1 | tail -3
timeout 300 python tools/time_pair.py --n 512 --angles 360 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/g53_c3.json 2> gpurun_out/g53_c3.err
timeout 900 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g53_c4.json 2> gpurun_out/g53_c4.err
timeout 600 python bench.py --angles 45 --solver lsqr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g53_45.json 2>&1
python - <<'P'
import json
for f in ["g53_c3", "g53_c4", "g53_45"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("kernels_ms"), d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
P
