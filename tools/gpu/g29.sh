timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
CTK_BP_VCHUNKS=1 timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
CTK_BP_VCHUNKS=4 timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
timeout 300 python tools/time_bp.py --n 128 --angles 100 --reps 9
CTK_BP_VCHUNKS=1 timeout 300 python tools/time_bp.py --n 128 --angles 100 --reps 9
timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_siddon.py tests/test_gpu_solvers.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "not c3 and not c4 and not c5" 2>&1 | tail -3
timeout 600 python bench.py --config C1 --steps 100 --no-cpu-baseline > gpurun_out/bench_c1b.json 2> gpurun_out/bench_c1b.err; tail -c 400 gpurun_out/bench_c1b.json
