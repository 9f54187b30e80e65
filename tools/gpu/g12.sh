timeout 300 python tools/dbg_sid.py 512 360 joseph atb 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_siddon.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/time_ops.py --n 256 --angles 180 2>&1 | head -2
timeout 600 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_C2b.json 2> gpurun_out/bench_C2b.err; tail -c 300 gpurun_out/bench_C2b.json
