# whole-slab pairing tests, chunk sweep for the pair, then C5 with the pair
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fwd_pair.py -x -q 2>&1 | tail -2
bash tools/gpu/g57.sh
timeout 2900 python bench.py --config C5 --steps 1 --warmup 3 > gpurun_out/g58_c5.json 2> gpurun_out/g58_c5.err; tail -c 300 gpurun_out/g58_c5.err
python - <<'P'
import json
d = json.loads(open("gpurun_out/g58_c5.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("kernels_ms"), d["clocks"]["reasons"], d.get("device_mem_used_gib"))
P
