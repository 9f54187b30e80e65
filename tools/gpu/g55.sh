# full GPU suite + smoke + C1 / C5 bench lines after the cgls reorder
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/g55_tests.log 2>&1; tail -3 gpurun_out/g55_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --config C1 --steps 3 --warmup 3 > gpurun_out/g55_c1.json 2> gpurun_out/g55_c1.err
timeout 1500 python bench.py --config C5 --steps 1 --warmup 3 > gpurun_out/g55_c5.json 2> gpurun_out/g55_c5.err
python - <<'P'
import json
for f in ["g55_c1", "g55_c5"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("e2e", {}).get("value"), d.get("kernels_ms"), d["clocks"]["reasons"], d.get("device_mem_used_gib"))
    except Exception as e:
        print(f, "ERR", e)
P
