# paired forward (ax2_f32): bitwise solver tests, then C3 / C4 with and without pairing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd_pair.py -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g50_c3_pair.json 2> gpurun_out/g50_c3_pair.err; tail -c 600 gpurun_out/g50_c3_pair.json
CTK_FWD_NO_PAIR=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g50_c3_nopair.json 2>&1; tail -c 600 gpurun_out/g50_c3_nopair.json
timeout 600 python bench.py --angles 45 --solver lsqr --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g50_45.json 2>&1; tail -c 400 gpurun_out/g50_45.json
python - <<'P'
import json
for f in ["g50_c3_pair", "g50_c3_nopair", "g50_45"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("kernels_ms"))
    except Exception as e:
        print(f, "ERR", e)
P
